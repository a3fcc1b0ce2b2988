"""Policy oracle: naive restatements of the reference's cache / cutoff / top-k
/ prefetch-task semantics — TEST INFRASTRUCTURE ONLY.

Each function follows a reference anchor and is pinned against golden
vectors generated from ``moesim`` itself (tests/golden/make_golden.py):

* :func:`topk` — trace.top_k_indices (trace.py:28-37): sort by (-score,
  index);
* :class:`NaiveLRU` — cache.ExpertCache (cache.py:34-143): a plain list in
  recency order with linear scans;
* :func:`brute_force_cutoff` — cutoff.solve_cutoff (cutoff.py:111-139) by
  exhaustive evaluation of both constraints at every L;
* :class:`PrefetchReplay` — the engine's Algorithm-2 pop-time semantics
  (enqueue_critical + worker_step re-check,
  prefetch.py:118-223; on_demand_load prefetch.py:276-301; verify lookups in
  ascending expert order simcore.py:368-372) replayed over recorded predictor
  outputs, including the slot each insert lands in (lowest free slot after
  the victims release theirs).
"""

from __future__ import annotations


def topk(scores, k):
    n = len(scores)
    if k > n:
        raise ValueError("k too large")
    return tuple(sorted(range(n), key=lambda i: (-scores[i], i))[:k])


class CacheErr(Exception):
    pass


class NaiveLRU:
    def __init__(self, capacity):
        self.capacity = capacity
        self.order = []  # least recent first
        self.pinned = set()
        self.slot = {}
        self.free = list(range(capacity))
        self.hits = self.misses = self.evictions = 0
        self.prefetch_evictions = self.prefetch_insertions = self.demand_insertions = 0

    # reference API -----------------------------------------------------
    def lookup(self, eid, touch):
        eid = tuple(eid)
        hit = eid in self.order
        if touch:
            if hit:
                self.hits += 1
                self.order.remove(eid)
                self.order.append(eid)
            else:
                self.misses += 1
        return hit

    def insert_batch(self, ids, kind="prefetch"):
        from paper_2510_10302_b200.cache import CacheError  # error class of the API under test

        kind = getattr(kind, "value", kind)
        batch = []
        for e in ids:
            e = tuple(e)
            if e not in batch:
                batch.append(e)
        if len(batch) > self.capacity - len(self.pinned):
            raise CacheError("too large")
        new = [e for e in batch if e not in self.order]
        overflow = max(0, len(self.order) + len(new) - self.capacity)
        victims = []
        for e in self.order:
            if len(victims) == overflow:
                break
            if e in self.pinned or e in batch:
                continue
            victims.append(e)
        if len(victims) < overflow:
            raise CacheError("not enough evictable")
        for v in victims:
            self.order.remove(v)
            self.free.append(self.slot.pop(v))
        self.free.sort()
        self.evictions += len(victims)
        if kind == "prefetch":
            self.prefetch_evictions += len(victims)
            self.prefetch_insertions += len(new)
        else:
            self.demand_insertions += len(new)
        for e in batch:
            if e in self.order:
                self.order.remove(e)
            else:
                self.slot[e] = self.free.pop(0)
            self.order.append(e)
        return victims

    def pin(self, ids):
        from paper_2510_10302_b200.cache import CacheError

        for e in ids:
            if tuple(e) not in self.order:
                raise CacheError("pin non-resident")
            self.pinned.add(tuple(e))

    def unpin(self, ids):
        for e in ids:
            self.pinned.discard(tuple(e))

    @property
    def lru_order(self):
        return list(self.order)

    def hit_rate(self):
        n = self.hits + self.misses
        return self.hits / n if n else 0.0

    def eviction_rate(self):
        return self.prefetch_evictions / self.prefetch_insertions if self.prefetch_insertions else 0.0


def brute_force_cutoff(inp):
    best = None
    for L in range(inp.l_all):
        n = (L + 1) * inp.k
        mem = inp.m_peak + n * inp.m_expert < inp.m_gpu
        lhs = max((L - 1) * inp.t_comp + inp.k * inp.t_io, n * inp.t_io)
        if mem and lhs <= inp.l_all * inp.t_comp:
            best = L
    return best


class PrefetchReplay:
    """Expected cache behaviour of the engine for recorded predictor outputs.

    Events, in program order:
      ("task", layer, [expert ids])   a predictor task popped by the worker
      ("verify", layer, [routed ids]) verify-stage lookups + demand load
    Produces the transfer list [(kind, layer, experts, slots)] and the final
    LRU order / counters.
    """

    def __init__(self, capacity):
        self.c = NaiveLRU(capacity)
        self.transfers = []
        self.tasks_completed = 0

    def task(self, layer, experts):
        load = []
        for e in experts:
            if e < 0:
                continue
            eid = (layer, int(e))
            if eid not in self.c.order and eid not in load:
                load.append(eid)
        if not load:
            return
        self.c.insert_batch(load, "prefetch")
        self.tasks_completed += 1
        self.transfers.append(("prefetch", layer, [e for _, e in load], [self.c.slot[x] for x in load]))

    def verify(self, layer, routed):
        required = sorted(set(int(e) for e in routed))
        missing = [(layer, e) for e in required if not self.c.lookup((layer, e), touch=True)]
        if missing:
            self.c.insert_batch(missing, "demand")
            self.transfers.append(("on_demand", layer, [e for _, e in missing], [self.c.slot[x] for x in missing]))
        return required
