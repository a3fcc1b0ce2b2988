"""Expert cache with LRU replacement (drop-in for moesim.cache).

Two implementations with one contract (``cache.py:34-143`` of the reference):

* :class:`ExpertCache` — pure-Python metadata cache (used by the API and the
  policy tests);
* :class:`NativeExpertCache` — the same contract over the native runtime
  (``spmoe_rt_*`` in ``libspmoe.so``) that owns the HBM slot table, the copy
  stream and the prefetch worker thread; this is what the B200 engine runs.

Contract: residents form a recency queue (head = least recently used);
``lookup(touch=True)`` counts a hit or miss and refreshes a hit;
``insert_batch`` evicts head-first, skipping pinned entries and members of the
batch, exactly enough to fit the genuinely new ids, then moves every member
to the tail in argument order; pinning a non-resident raises ``CacheError``.
"""

from __future__ import annotations

import ctypes as C
import enum
from collections import OrderedDict
from typing import Iterable, NamedTuple


class ExpertId(NamedTuple):
    layer: int
    expert: int


class InsertKind(str, enum.Enum):
    PREFETCH = "prefetch"
    DEMAND = "demand"


class CacheError(Exception):
    """Contract violation: over-large batch or pinning a non-resident."""


class _Counters:
    def reset_stats(self) -> None:
        self.hits = 0
        self.misses = 0
        self.evictions = 0
        self.prefetch_evictions = 0
        self.prefetch_insertions = 0
        self.demand_insertions = 0

    def eviction_rate(self) -> float:
        """Prefetch-caused evictions per prefetch insertion (0/0 -> 0)."""
        return self.prefetch_evictions / self.prefetch_insertions if self.prefetch_insertions else 0.0

    def hit_rate(self) -> float:
        n = self.hits + self.misses
        return self.hits / n if n else 0.0


class ExpertCache(_Counters):
    """Metadata-only LRU cache of ``ExpertId`` (the reference semantics)."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = capacity
        self._lru: OrderedDict[ExpertId, None] = OrderedDict()
        self.pinned: set[ExpertId] = set()
        self.reset_stats()

    def __len__(self) -> int:
        return len(self._lru)

    def __contains__(self, expert_id) -> bool:
        return expert_id in self._lru

    @property
    def lru_order(self) -> list[ExpertId]:
        return list(self._lru)

    def lookup(self, expert_id: ExpertId, touch: bool) -> bool:
        present = expert_id in self._lru
        if not touch:
            return present
        if present:
            self.hits += 1
            self._lru.move_to_end(expert_id)
        else:
            self.misses += 1
        return present

    def insert_batch(self, ids: Iterable[ExpertId], kind: InsertKind = InsertKind.PREFETCH) -> list[ExpertId]:
        members = list(OrderedDict.fromkeys(ids))
        room = self.capacity - len(self.pinned)
        if len(members) > room:
            raise CacheError(f"batch of {len(members)} exceeds evictable capacity {room}")
        member_set = set(members)
        fresh = [m for m in members if m not in self._lru]
        need = len(self._lru) + len(fresh) - self.capacity
        victims: list[ExpertId] = []
        if need > 0:
            candidates = (e for e in self._lru if e not in self.pinned and e not in member_set)
            for e in candidates:
                victims.append(e)
                if len(victims) == need:
                    break
            if len(victims) < need:
                raise CacheError("not enough evictable entries for batch insert")
            for v in victims:
                del self._lru[v]
        self.evictions += len(victims)
        if kind is InsertKind.PREFETCH:
            self.prefetch_evictions += len(victims)
            self.prefetch_insertions += len(fresh)
        else:
            self.demand_insertions += len(fresh)
        for m in members:
            self._lru[m] = None
            self._lru.move_to_end(m)
        return victims

    def pin(self, ids: Iterable[ExpertId]) -> None:
        for e in ids:
            if e not in self._lru:
                raise CacheError(f"cannot pin non-resident expert {e}")
            self.pinned.add(e)

    def unpin(self, ids: Iterable[ExpertId]) -> None:
        for e in ids:
            self.pinned.discard(e)


_KIND = {InsertKind.PREFETCH: 0, InsertKind.DEMAND: 1}


class NativeExpertCache:
    """The cache contract over the native slot-table runtime.

    Besides the reference API it exposes the slot of each resident expert,
    demand loads that copy into HBM, per-slot copy/read events and the
    asynchronous prefetch worker (Algorithm 2).
    """

    COUNTER_NAMES = (
        "hits",
        "misses",
        "evictions",
        "prefetch_evictions",
        "prefetch_insertions",
        "demand_insertions",
        "tasks_completed",
        "tasks_aborted",
        "prefetch_bytes",
        "demand_bytes",
        "n_resident",
        "evictions_of_queued_targets",
        "handoff_timeouts",
    )

    def __init__(
        self,
        capacity: int,
        num_layers: int,
        num_experts: int,
        *,
        dev_pool_ptr: int = 0,
        host_pool_ptr: int = 0,
        host_index=None,
        slot_bytes: int = 0,
        copy_stream_ptr: int = 0,
        batched_io: bool = True,
    ):
        from . import _native

        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self._lib = _native.load()
        hidx = None
        if host_index is not None:
            hidx = (C.c_int32 * (num_layers * num_experts))(*[int(v) for v in host_index])
        self._hidx = hidx
        h = self._lib.spmoe_rt_create(
            capacity,
            num_layers,
            num_experts,
            dev_pool_ptr or None,
            host_pool_ptr or None,
            hidx,
            slot_bytes,
            copy_stream_ptr or None,
            1 if batched_io else 0,
        )
        if not h:
            raise CacheError("spmoe_rt_create failed")
        self._h = h
        self.capacity = capacity
        self.num_layers = num_layers
        self.num_experts = num_experts

    # -- lifecycle ------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.spmoe_rt_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    # -- reference API ------------------------------------------------------
    @staticmethod
    def _arrays(ids):
        ids = [ExpertId(*e) for e in ids]
        n = len(ids)
        L = (C.c_int32 * max(n, 1))(*[e.layer for e in ids])
        X = (C.c_int32 * max(n, 1))(*[e.expert for e in ids])
        return ids, n, L, X

    def lookup(self, expert_id: ExpertId, touch: bool) -> bool:
        return bool(self._lib.spmoe_rt_lookup(self._h, expert_id[0], expert_id[1], 1 if touch else 0))

    def __contains__(self, expert_id) -> bool:
        return self.lookup(ExpertId(*expert_id), touch=False)

    def __len__(self) -> int:
        return self.counters()["n_resident"]

    def insert_batch(self, ids: Iterable[ExpertId], kind: InsertKind = InsertKind.PREFETCH) -> list[ExpertId]:
        ids, n, L, X = self._arrays(ids)
        out = (C.c_int32 * max(2 * n, 2))()
        nv = self._lib.spmoe_rt_insert_batch(self._h, L, X, n, _KIND[InsertKind(kind)], out)
        if nv < 0:
            raise CacheError("batch exceeds evictable capacity or not enough evictable entries")
        return [ExpertId(out[2 * i], out[2 * i + 1]) for i in range(nv)]

    def pin(self, ids: Iterable[ExpertId]) -> None:
        ids, n, L, X = self._arrays(ids)
        if self._lib.spmoe_rt_pin(self._h, L, X, n) != 0:
            raise CacheError("cannot pin non-resident expert")

    def unpin(self, ids: Iterable[ExpertId]) -> None:
        ids, n, L, X = self._arrays(ids)
        self._lib.spmoe_rt_unpin(self._h, L, X, n)

    @property
    def lru_order(self) -> list[ExpertId]:
        cap = self.capacity
        L = (C.c_int32 * cap)()
        X = (C.c_int32 * cap)()
        n = self._lib.spmoe_rt_lru_order(self._h, L, X, cap)
        return [ExpertId(L[i], X[i]) for i in range(n)]

    def counters(self) -> dict[str, int]:
        buf = (C.c_int64 * len(self.COUNTER_NAMES))()
        self._lib.spmoe_rt_counters(self._h, buf)
        return dict(zip(self.COUNTER_NAMES, list(buf)))

    def __getattr__(self, name):
        if name in NativeExpertCache.COUNTER_NAMES:
            return self.counters()[name]
        raise AttributeError(name)

    def reset_stats(self) -> None:
        self._lib.spmoe_rt_reset_stats(self._h)

    def eviction_rate(self) -> float:
        c = self.counters()
        return c["prefetch_evictions"] / c["prefetch_insertions"] if c["prefetch_insertions"] else 0.0

    def hit_rate(self) -> float:
        c = self.counters()
        n = c["hits"] + c["misses"]
        return c["hits"] / n if n else 0.0

    # -- device-side extensions -------------------------------------------
    def slot_of(self, layer: int, expert: int) -> int:
        return self._lib.spmoe_rt_slot_of(self._h, layer, expert)

    def demand_load(self, ids) -> list[int]:
        """Insert the non-resident ids as one DEMAND batch and copy them on the
        copy stream; returns the slot of every id."""
        from . import _native

        ids, n, L, X = self._arrays(ids)
        slots = (C.c_int32 * max(n, 1))()
        st = self._lib.spmoe_rt_demand_load(self._h, L, X, n, slots)
        if st == -1:
            raise CacheError("demand batch exceeds evictable capacity")
        _native.check("spmoe_rt_demand_load", st)
        return [slots[i] for i in range(n)]

    def wait_slot(self, slot: int, stream_ptr: int) -> None:
        from . import _native

        _native.check("spmoe_rt_wait_slot", self._lib.spmoe_rt_wait_slot(self._h, slot, stream_ptr))

    def mark_read(self, slot: int, stream_ptr: int) -> None:
        from . import _native

        _native.check("spmoe_rt_mark_read", self._lib.spmoe_rt_mark_read(self._h, slot, stream_ptr))

    def slot_ready(self, slot: int) -> bool:
        return bool(self._lib.spmoe_rt_slot_ready(self._h, slot))

    # -- prefetch worker ----------------------------------------------------
    def start_worker(self) -> None:
        self._lib.spmoe_rt_worker_start(self._h)

    def stop_worker(self) -> None:
        self._lib.spmoe_rt_worker_stop(self._h)

    def push_task(self, layer: int, host_idx_ptr: int, k: int, ready_event_ptr: int, issue_token: int = -1) -> None:
        from . import _native

        _native.check(
            "spmoe_rt_push_task",
            self._lib.spmoe_rt_push_task(self._h, layer, host_idx_ptr, k, ready_event_ptr or None, issue_token),
        )

    def drain(self) -> None:
        """Wait for every pushed task; raises if a copy, event wait or flag
        hand-off failed since the last drain (the failed task's experts are
        not left resident)."""
        from . import _native

        _native.check("spmoe_rt_drain", self._lib.spmoe_rt_drain(self._h))

    def abort_pending(self) -> int:
        return self._lib.spmoe_rt_abort_pending(self._h)

    def transfer_log(self, cap: int = 1 << 16):
        rec = (C.c_int32 * (4 * cap))()
        t = (C.c_double * (2 * cap))()
        n = self._lib.spmoe_rt_transfer_log(self._h, rec, t, cap)
        out = []
        for i in range(n):
            ex = (C.c_int32 * 256)()
            ne = self._lib.spmoe_rt_transfer_experts(self._h, i, ex, 256)
            out.append(
                {
                    "layer": rec[4 * i],
                    "n_experts": rec[4 * i + 1],
                    "kind": "prefetch" if rec[4 * i + 2] == 0 else "on_demand",
                    "seq": rec[4 * i + 3],
                    "start_ms": t[2 * i],
                    "end_ms": t[2 * i + 1],
                    "experts": tuple(ex[j] for j in range(ne)),
                    "wire_bytes": int(self._lib.spmoe_rt_transfer_wire_bytes(self._h, i)),
                    "copy_end_ms": float(self._lib.spmoe_rt_transfer_copy_end_ms(self._h, i)),
                }
            )
        return out

    def set_codec(self, row_stride: int, staging_ptr: int, staging_bytes: int, n_staging: int,
                  decode_stream_ptr: int) -> None:
        """Host rows are XC blobs from now on (spmoe_rt_set_codec)."""
        from . import _native

        _native.check("spmoe_rt_set_codec", self._lib.spmoe_rt_set_codec(
            self._h, row_stride, staging_ptr, staging_bytes, n_staging, decode_stream_ptr))

    def decode_timing(self, enable) -> None:
        """Time every XC segment decode from now on (profiling): ``"device"``
        (or 2) records each launch's device-clock span (globaltimer, first
        CTA start -> last CTA end), ``True`` / ``"events"`` (or 1) brackets it
        with CUDA events on the decode stream, falsy stops."""
        from . import _native

        if isinstance(enable, str):
            mode = {"device": 2, "events": 1}[enable]
        else:
            mode = 1 if enable is True else int(enable or 0)
        _native.check("spmoe_rt_decode_timing", self._lib.spmoe_rt_decode_timing(self._h, mode))

    def decode_stats(self) -> dict:
        """Timed decodes since the last call: total ms, bytes read + written,
        launches, achieved GB/s."""
        ms, b, n = C.c_double(), C.c_int64(), C.c_int64()
        self._lib.spmoe_rt_decode_stats(self._h, C.byref(ms), C.byref(b), C.byref(n))
        return {"ms": ms.value, "bytes": b.value, "launches": n.value,
                "gbs": (b.value / (ms.value / 1e3) / 1e9) if ms.value > 0 else None}

    def wire_bytes(self) -> dict[str, int]:
        """Bytes that crossed the host link since the last reset."""
        o = (C.c_int64 * 2)()
        self._lib.spmoe_rt_wire_bytes(self._h, o)
        return {"prefetch": int(o[0]), "demand": int(o[1])}

    def clear_log(self) -> None:
        self._lib.spmoe_rt_clear_log(self._h)

    def since_epoch_ms(self, event) -> float:
        """ms from the runtime epoch to a recorded torch.cuda.Event (timing)."""
        return float(self._lib.spmoe_rt_since_epoch_ms(self._h, event.cuda_event))
