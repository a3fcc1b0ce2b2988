"""Expert-parallel verify MoE (SURVEY.md §8 row e, the optional mode).

The reference has no expert parallelism (it simulates one device,
``simcore.py:182-515``); this is the B200 multi-GPU variant of the verify
MoE layer (Eq. 1): the routed experts of every layer are split into
contiguous blocks, rank r owning ``[lo_r, hi_r)``, and each verify layer does

    K1 route (local tokens) -> K2 permute (expert order = owner order)
    -> all-gather per-expert counts -> gather rows -> all-to-all dispatch
    -> K2/K3 on the received rows with the rank's own expert slots
    -> gather back to receive order -> all-to-all combine
    -> K4 weighted combine + residual (K2's inverse map indexes the returned
       rows directly, because the send order IS K2's permuted order).

With the draft_prefetch policy each rank drafts its own stream and runs
Algorithm 1's predictor (K1) on it; the predicted expert ids of every
(draft step, layer <= cutoff) are all-gathered on the host (a gloo group
beside the NCCL one, E-sized int vectors) and each rank enqueues the union
of every rank's predictions that it OWNS (rank order, then token order,
first occurrence) into its own prefetch worker: the owner's cache is the one
the verify will read, whichever stream's draft predicted the expert.

Because expert ids are contiguous per owner, K2's stable expert order is
already grouped by destination rank: no extra sort, the send counts are
prefix sums of the per-expert counts the host already holds for its cache
decisions.  One process per GPU; the collectives go through
``torch.distributed`` (NCCL over NVLink on a GPU box, gloo in the CPU tests,
where ``gather`` is injected).  World size 1 degenerates to local copies.
"""

from __future__ import annotations

from typing import Callable

import numpy as np
import torch


def shard_range(num_experts: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced expert block ``[lo, hi)`` owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    if num_experts < world:
        raise ValueError(f"expert parallelism needs experts_per_layer ({num_experts}) >= world size ({world})")
    return rank * num_experts // world, (rank + 1) * num_experts // world


def owner_table(num_experts: int, world: int) -> np.ndarray:
    """``owner[e]`` = the rank hosting routed expert e."""
    own = np.empty(num_experts, dtype=np.int64)
    for r in range(world):
        lo, hi = shard_range(num_experts, r, world)
        own[lo:hi] = r
    return own


def send_counts_of(counts: np.ndarray, world: int) -> list[int]:
    """Rows sent to each rank from per-expert routed counts (K2 order)."""
    E = counts.shape[0]
    return [int(counts[slice(*shard_range(E, r, world))].sum()) for r in range(world)]


def owned_predictions(all_idx: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """The experts in ``[lo, hi)`` among every rank's predicted ids
    (``all_idx [world, n]``, -1 = none), in rank order then token order,
    each once (first occurrence)."""
    out, seen = [], set()
    for e in np.asarray(all_idx).reshape(-1):
        e = int(e)
        if lo <= e < hi and e not in seen:
            seen.add(e)
            out.append(e)
    return np.asarray(out, dtype=np.int32)


def _default_gather(src: torch.Tensor, idx: torch.Tensor, div: int, out: torch.Tensor | None = None):
    from .kernels import gather_rows

    return gather_rows(src, idx, div, out=out)


class ExpertParallelExchange:
    """The two all-to-alls of one expert-parallel MoE layer.

    ``dispatch(x, perm_token, counts)`` sends each routed (token, choice)
    row to the owner of its expert and returns the received rows and their
    global expert ids (device and host copies), derived from the all-gathered
    per-expert counts.  ``combine(y_recv)`` sends
    the expert outputs back; the result is ``[T*k, H]`` in the sender's K2
    permuted order, ready for K4 with K2's inverse map.
    """

    def __init__(self, num_experts: int, top_k: int, group=None,
                 gather: Callable | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        # without a process group the exchange is a local copy (world 1)
        self.local_only = not dist.is_initialized()
        self.world = 1 if self.local_only else dist.get_world_size(group)
        self.rank = 0 if self.local_only else dist.get_rank(group)
        self.E, self.k = num_experts, top_k
        self.lo, self.hi = shard_range(num_experts, self.rank, self.world)
        self.gather = gather or _default_gather
        # host-side exchanges (predicted experts) go through a CPU group: the
        # NCCL group itself when it is gloo, else a gloo group of the same ranks
        self.host_group = None
        if not self.local_only:
            ranks = dist.get_process_group_ranks(group) if group is not None else list(range(dist.get_world_size()))
            self.host_group = group if dist.get_backend(group) == "gloo" else dist.new_group(ranks=ranks, backend="gloo")
        self._send: list[int] = []
        self._recv: list[int] = []
        self.bytes_sent = 0

    @property
    def local_experts(self) -> range:
        return range(self.lo, self.hi)

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits) -> None:
        if self.local_only:
            out.copy_(inp)
            return
        self.dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def _all_counts(self, counts: np.ndarray, device) -> np.ndarray:
        """Every rank's per-expert routed counts ``[world, E]`` (one
        all-gather of E ints): gives both exchange splits and the expert id
        of every received row without sending ids."""
        counts = np.asarray(counts, dtype=np.int64).reshape(1, -1)
        if self.local_only:
            return counts
        # NCCL needs device tensors; gloo host tensors
        dev = device if self.dist.get_backend(self.group) == "nccl" else "cpu"
        mine = torch.from_numpy(counts.copy()).to(dev)
        allc = torch.empty((self.world, counts.shape[1]), dtype=torch.int64, device=dev)
        self.dist.all_gather_into_tensor(allc, mine, group=self.group)
        return allc.cpu().numpy()

    def gather_predictions(self, idx: np.ndarray) -> np.ndarray:
        """Every rank's predicted expert ids for one (draft step, layer):
        ``[world, n]`` host int32 (equal n on every rank)."""
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int32).reshape(1, -1))
        if self.local_only:
            return idx
        mine = torch.from_numpy(idx.copy())
        parts = [torch.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(parts, mine, group=self.host_group)
        return torch.cat(parts, dim=0).numpy()

    def agree(self, value: int | None) -> int | None:
        """Rank 0's value on every rank (None travels as -1): the predictor
        exchange runs once per (draft step, layer <= cutoff), so every rank
        must use the same cutoff even when their measured timings differ."""
        if self.local_only:
            return value
        t = torch.tensor([-1 if value is None else int(value)], dtype=torch.int64)
        self.dist.broadcast(t, src=self.dist.get_global_rank(self.host_group, 0) if self.group is not None else 0,
                            group=self.host_group)
        v = int(t.item())
        return None if v < 0 else v

    def prefetch_share(self, idx: np.ndarray) -> np.ndarray:
        """This rank's experts among all ranks' predictions (see module doc)."""
        return owned_predictions(self.gather_predictions(idx), self.lo, self.hi)

    def dispatch(self, x: torch.Tensor, perm_token: torch.Tensor, counts: np.ndarray):
        """x ``[T, H]``; perm_token = K2's ``perm_token`` (the token of every
        permuted row, rows grouped by expert ascending); counts = routed rows
        per expert (host).  Returns ``(x_recv [R, H], e_recv [R] int32,
        e_recv_host np.ndarray)``; received rows are grouped by sender rank,
        then by expert ascending."""
        T, H = x.shape
        n = T * self.k
        counts = np.asarray(counts, dtype=np.int64)
        if int(counts.sum()) != n:
            raise ValueError("per-expert counts do not cover the routed rows")
        allc = self._all_counts(counts, x.device)
        self._send = send_counts_of(counts, self.world)
        self._recv = [int(allc[s, self.lo:self.hi].sum()) for s in range(self.world)]
        R = sum(self._recv)
        x_send = self.gather(x, perm_token[:n], 1)
        x_recv = torch.empty((R, H), dtype=x.dtype, device=x.device)
        self._a2a(x_recv, x_send, self._recv, self._send)
        local = np.arange(self.lo, self.hi, dtype=np.int32)
        e_host = np.concatenate([np.repeat(local, allc[s, self.lo:self.hi]) for s in range(self.world)]
                                ).astype(np.int32) if R else np.zeros((0,), np.int32)
        e_recv = torch.from_numpy(e_host).to(x.device)
        self.bytes_sent += (n - self._send[self.rank]) * H * x.element_size()
        return x_recv, e_recv, e_host

    def combine(self, y_recv: torch.Tensor) -> torch.Tensor:
        """y_recv ``[R, H]`` in receive order -> ``[T*k, H]`` in send order."""
        n = sum(self._send)
        out = torch.empty((n,) + tuple(y_recv.shape[1:]), dtype=y_recv.dtype, device=y_recv.device)
        self._a2a(out, y_recv, self._send, self._recv)
        return out
