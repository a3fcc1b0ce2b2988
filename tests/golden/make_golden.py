"""Generate golden fixtures from the reference package ``moesim``.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/moesim_golden.json.  The fixtures pin the policy half of
the hot path to the reference's own behaviour:
top-k ordering incl. ties (trace.py:28-37 / predictor.py:100-106), the LRU
cache contract under random operation sequences (cache.py:62-122), the
cutoff solver (cutoff.py:111-170) on random inputs and on the shipped
configs, and config parsing of the shipped YAML files (config.py:315-405).
"""

from __future__ import annotations

import json
import random
import sys
from dataclasses import asdict
from pathlib import Path

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

import moesim  # noqa: E402
from moesim.cache import CacheError, ExpertCache, ExpertId, InsertKind  # noqa: E402
from moesim.cutoff import CutoffInput, cutoff_input_from_specs, feasibility_report, solve_cutoff  # noqa: E402
from moesim.trace import top_k_indices  # noqa: E402


def gen_topk(rng):
    cases = [
        ([0.1, 0.4, 0.4, 0.1], 2),  # test_trace.py:41-43 known answer (1, 2)
        ([0.25] * 4, 2),  # all-tie -> (0, 1)
        ([0.0] * 8, 3),
        ([1.0, 1.0, 0.5, 1.0], 3),
    ]
    for _ in range(300):
        E = rng.choice([8, 16, 60, 64])
        k = rng.randint(1, min(8, E))
        if rng.random() < 0.5:
            # quantised scores -> many exact ties
            scores = [rng.randint(0, 5) / 4.0 for _ in range(E)]
        else:
            scores = [rng.random() for _ in range(E)]
        cases.append((scores, k))
    return [{"scores": s, "k": k, "expected": list(top_k_indices(s, k))} for s, k in cases]


def gen_cache(rng):
    seqs = []
    for trial in range(40):
        cap = rng.randint(1, 12)
        c = ExpertCache(cap)
        ops = []
        for _ in range(300):
            r = rng.random()
            if r < 0.45:
                eid = (rng.randrange(4), rng.randrange(16))
                touch = rng.random() < 0.7
                hit = c.lookup(ExpertId(*eid), touch=touch)
                ops.append({"op": "lookup", "id": eid, "touch": touch, "ret": hit})
            elif r < 0.85:
                n = rng.randint(1, 4)
                ids = [(rng.randrange(4), rng.randrange(16)) for _ in range(n)]
                kind = "prefetch" if rng.random() < 0.5 else "demand"
                try:
                    v = c.insert_batch([ExpertId(*e) for e in ids], InsertKind(kind))
                    ops.append({"op": "insert", "ids": ids, "kind": kind, "ret": [list(x) for x in v]})
                except CacheError:
                    ops.append({"op": "insert", "ids": ids, "kind": kind, "ret": "CacheError"})
            elif r < 0.93:
                order = c.lru_order
                if order and rng.random() < 0.8:
                    e = order[rng.randrange(len(order))]
                    c.pin([e])
                    ops.append({"op": "pin", "ids": [list(e)], "ret": None})
                else:
                    e = (rng.randrange(4), rng.randrange(16))
                    try:
                        c.pin([ExpertId(*e)])
                        ops.append({"op": "pin", "ids": [list(e)], "ret": None})
                    except CacheError:
                        ops.append({"op": "pin", "ids": [list(e)], "ret": "CacheError"})
            else:
                pins = list(c.pinned)
                if pins:
                    e = pins[rng.randrange(len(pins))]
                    c.unpin([e])
                    ops.append({"op": "unpin", "ids": [list(e)], "ret": None})
        seqs.append(
            {
                "capacity": cap,
                "ops": ops,
                "final_order": [list(e) for e in c.lru_order],
                "counters": {
                    "hits": c.hits, "misses": c.misses, "evictions": c.evictions,
                    "prefetch_evictions": c.prefetch_evictions,
                    "prefetch_insertions": c.prefetch_insertions,
                    "demand_insertions": c.demand_insertions,
                },
                "hit_rate": c.hit_rate(),
                "eviction_rate": c.eviction_rate(),
            }
        )
    # worked example of test_cache.py:157-165 in the same format
    return seqs


def gen_cutoff(rng):
    cases = []
    for _ in range(500):
        inp = CutoffInput(
            k=rng.randint(1, 6),
            l_all=rng.randint(1, 40),
            t_comp=rng.uniform(0.0001, 0.01),
            t_io=rng.uniform(0.0001, 0.03),
            m_expert=rng.randint(1_000_000, 400_000_000),
            m_gpu=24_000_000_000,
            m_peak=rng.randint(1_000_000_000, 23_000_000_000),
        )
        r = solve_cutoff(inp)
        L = rng.randrange(inp.l_all)
        fr = feasibility_report(inp, L)
        cases.append({"input": asdict(inp), "layer": r.layer, "n_expert": r.n_expert,
                      "binding": r.binding_constraint.value, "feasible": r.feasible,
                      "report_layer": L, "mem_slack": fr.memory_slack_bytes,
                      "overlap_slack": fr.overlap_slack_seconds})
    return cases


def gen_configs():
    out = {}
    for p in sorted((REF.parent / "configs").glob("*.yaml")):
        model, hw, timings, policy = moesim.load_config(p)
        res = solve_cutoff(cutoff_input_from_specs(model, hw, timings, policy.prefetch_k))
        out[p.name] = {
            "model": asdict(model),
            "hardware": asdict(hw),
            "timings": asdict(timings),
            "policy": {**asdict(policy), "policy": policy.policy.value},
            "cutoff": {"layer": res.layer, "n_expert": res.n_expert,
                       "binding": res.binding_constraint.value, "feasible": res.feasible},
            "capacity": moesim.cache_capacity_slots(model, hw, policy),
        }
    return out


def main():
    rng = random.Random(20251017)
    doc = {
        "generator": "tests/golden/make_golden.py",
        "reference": "moesim " + moesim.__version__ + " (/root/reference/pkg)",
        "numpy": np.__version__,
        "topk": gen_topk(rng),
        "cache": gen_cache(rng),
        "cutoff": gen_cutoff(rng),
        "configs": gen_configs(),
    }
    out = Path(__file__).resolve().parent / "moesim_golden.json"
    out.write_text(json.dumps(doc))
    print(out, out.stat().st_size)


if __name__ == "__main__":
    main()
