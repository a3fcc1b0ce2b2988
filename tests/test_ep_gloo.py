"""Expert-parallel exchange plumbing (ep.py) on CPU: world sizes 2 and 3 over
gloo (127.0.0.1).  Each rank routes its own tokens, dispatches rows to the
experts' owners, applies a per-expert function only to rows of experts it
owns, and combines; the result must equal applying every expert locally.
The row gather is injected as torch indexing (the product path uses the
CUDA ``spmoe_gather_rows`` kernel, covered by the GPU tests)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2510_10302_b200.ep import owner_table, send_counts_of, shard_range


def test_shard_ranges_partition():
    for E in (1, 2, 7, 8, 60, 64):
        for world in range(1, min(E, 9) + 1):
            rs = [shard_range(E, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == E
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in rs]
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
            own = owner_table(E, world)
            for r, (lo, hi) in enumerate(rs):
                assert (own[lo:hi] == r).all()
    with pytest.raises(ValueError):
        shard_range(4, 0, 5)


def test_send_counts():
    counts = np.array([3, 0, 1, 2, 5, 0, 0, 4])
    assert send_counts_of(counts, 1) == [15]
    assert send_counts_of(counts, 2) == [6, 9]
    assert send_counts_of(counts, 8) == list(counts)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather(src, idx, div, out=None):
    return src[idx.long() // div].clone()


def _expert_fn(x: torch.Tensor, e: torch.Tensor) -> torch.Tensor:
    # distinct per-expert affine map (float64, exact enough to compare ==)
    e = e.to(torch.float64).unsqueeze(1)
    return x.to(torch.float64) * (e + 1.0) + 0.25 * e


def _worker(rank, world, port, q, E, k, H, T_of_rank):
    import torch.distributed as dist

    from paper_2510_10302_b200.ep import ExpertParallelExchange

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = ExpertParallelExchange(E, k, gather=_gather)
        rng = np.random.default_rng(100 + rank)
        ok = True
        for it in range(6):
            T = T_of_rank[(rank + it) % len(T_of_rank)]
            x = torch.from_numpy(rng.standard_normal((T, H))).to(torch.float32)
            if it == 3:  # every token of this rank to one expert (max imbalance)
                idx = np.zeros((T, k), dtype=np.int32) + (E - 1)
                if k > 1:
                    idx[:, 1:] = np.arange(k - 1, dtype=np.int32)
            else:
                idx = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32) \
                    if T else np.zeros((0, k), dtype=np.int32)
            flat = idx.reshape(-1)
            perm = np.argsort(flat, kind="stable").astype(np.int32)  # K2's expert order
            counts = np.bincount(flat, minlength=E)
            # K2's perm_token: the token of every permuted row
            x_recv, e_recv, e_host = ex.dispatch(x, torch.from_numpy(perm // k), counts)
            assert x_recv.shape[0] == e_host.shape[0]
            assert ((e_host >= ex.lo) & (e_host < ex.hi)).all()
            y_recv = _expert_fn(x_recv, e_recv)
            y_back = ex.combine(y_recv)
            y = torch.empty_like(y_back)
            y[torch.from_numpy(perm).long()] = y_back  # row of flat (t, i)
            ref = _expert_fn(x.repeat_interleave(k, dim=0), torch.from_numpy(flat.copy()))
            ok &= bool(torch.equal(y, ref))
        q.put((rank, ok, ex.bytes_sent))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,E,k", [(2, 8, 2), (3, 60, 4), (2, 64, 6)])
def test_gloo_expert_parallel_exchange(world, E, k):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    T_of_rank = [5, 0, 1, 9]  # includes a rank with no tokens this layer
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, E, k, 16, T_of_rank)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert sum(b for *_, b in res) > 0


def test_owned_predictions_order_and_dedup():
    from paper_2510_10302_b200.ep import owned_predictions

    allidx = np.array([[3, 1, -1, 3], [0, 2, 1, 3]], dtype=np.int32)
    assert owned_predictions(allidx, 1, 4).tolist() == [3, 1, 2]  # rank order, token order, first occurrence
    assert owned_predictions(allidx, 0, 1).tolist() == [0]
    assert owned_predictions(allidx, 4, 8).size == 0
    assert owned_predictions(np.full((3, 2), -1), 0, 8).size == 0


def _pred_worker(rank, world, port, q, E, n):
    import torch.distributed as dist

    from paper_2510_10302_b200.ep import ExpertParallelExchange, owned_predictions

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = ExpertParallelExchange(E, 2, gather=_gather)
        ok = True
        for step in range(4):
            # every rank can reconstruct every rank's predictions from the seeds
            preds = [np.random.default_rng(1000 * step + r).integers(-1, E, size=n).astype(np.int32)
                     for r in range(world)]
            share = ex.prefetch_share(preds[rank])
            ok &= share.tolist() == owned_predictions(np.stack(preds), ex.lo, ex.hi).tolist()
            ok &= bool(((share >= ex.lo) & (share < ex.hi)).all())
        # every rank runs rank 0's cutoff (None travels too)
        ok &= ex.agree(3 + rank) == 3 and ex.agree(None if rank == 0 else 5) is None
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,E", [(2, 8), (3, 60)])
def test_gloo_prefetch_share(world, E):
    """EP draft_prefetch hand-off: each rank enqueues exactly the union of all
    ranks' predictions that it owns (ep.ExpertParallelExchange.prefetch_share),
    on the cutoff all ranks agreed on (rank 0's)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pred_worker, args=(r, world, port, q, E, 6)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
