"""BASELINE configs #3 / #4 sweeps on one B200 (one model build per arch):

  deepseek: DeepSeek-V2-Lite shapes, offload budget 25 %, cutoff-layer sweep
            (solver's choice + explicit 0..L-1) -> TPOT, hit rate, hidden
            prefetch fraction;
  qwen:     Qwen1.5-MoE-A2.7B shapes, draft length N in {2,4,8}, batch
            {1,2,4,8}, budget {12.5,25,50} % -> TPOT, tokens/s, hit rate;
  mixtral:  Mixtral-8x7B policy and cutoff points at 25 %;
  mixtral_grid: Mixtral-8x7B budget {12.5,25,50,100} %, N {2,8}, batch {2,4}.

python tools/sweeps.py deepseek|qwen|mixtral|mixtral_grid [--out profiles/sweeps_r1.jsonl] [--steps 6]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec  # noqa: E402
from paper_2510_10302_b200.calibrate import b200_timings  # noqa: E402
from paper_2510_10302_b200.engine import SpecMoEEngine  # noqa: E402
from paper_2510_10302_b200.model import get_arch  # noqa: E402


def point(arch, hw, state, *, N=4, batch=1, budget=0.25, cutoff=None, policy="draft_prefetch", steps=6, warmup=2,
          window=True, ffn_impl="cuda_core"):
    E_all = arch.num_layers * arch.num_experts
    cap = max(arch.num_experts, int(round(budget * E_all)))
    pk = 1 if arch.num_experts <= 16 else arch.top_k
    pol = PolicySpec(policy=Policy(policy), prefetch_k=pk, draft_length=N, acceptance_rate=1.0, seed=1234,
                     cutoff_layer=cutoff, cache_capacity_experts=cap)
    eng = SpecMoEEngine(arch, hw, b200_timings(arch, hw), pol, batch=batch, max_tokens=64 + (steps + warmup + 2) * (N + 1),
                        window_tokens=N if window else 1, model_state=state, ffn_impl=ffn_impl)
    try:
        g = torch.Generator().manual_seed(1000)
        eng.prefill(torch.randint(0, arch.vocab, (batch, 64), generator=g))
        for _ in range(warmup):
            eng.step()
        torch.cuda.synchronize()
        eng._reset_run_state()
        eng.cache.reset_stats()
        eng.cache.clear_log()
        for _ in range(steps):
            eng.step()
        rep = eng.report()
        ex = rep.extras
        return {
            "arch": arch.name, "N": N, "batch": batch, "budget": budget, "capacity": cap, "policy": policy,
            "cutoff": rep.cutoff_effective, "tpot_ms": rep.tpot * 1e3, "tokens_per_s": ex["tokens_per_s"],
            "hit_rate": rep.hit_rate, "acceptance": ex["acceptance_rate"],
            "hidden_prefetch_fraction": ex["hidden_prefetch_fraction"], "h2d_gbs": ex["h2d_gbs"],
            "breakdown": rep.latency_breakdown, "prefetch_insertions": rep.counters["prefetch_insertions"],
            "demand_insertions": rep.counters["demand_insertions"],
            "ms_per_iteration": rep.total_time * 1e3 / max(1, len(rep.iterations)),
            "ffn_impl": ffn_impl,
            "host_codec": ex.get("host_codec"), "wire_ratio": ex.get("h2d_wire_ratio"),
            "h2d_wire_gbs": ex.get("h2d_wire_gbs"),
        }
    finally:
        eng.close()


def facade(arch, hw, state, a):
    import paper_2510_10302_b200 as m
    from paper_2510_10302_b200.model import model_spec_for

    cap = max(arch.num_experts, int(round(0.25 * arch.num_layers * arch.num_experts)))
    pol = PolicySpec(policy=Policy.DRAFT_PREFETCH, prefetch_k=arch.top_k, draft_length=4, acceptance_rate=1.0,
                     seed=1234, cutoff_layer=0, cache_capacity_experts=cap)
    g = torch.Generator().manual_seed(1000)
    prompts = torch.randint(0, arch.vocab, (1, 64), generator=g)
    kw = dict(arch=arch, prompts=prompts, max_new_tokens=5 * a.steps, model_state=state, window_tokens=4)
    spec, t = model_spec_for(arch), b200_timings(arch, hw)

    def row(label, v, rep):
        r = {"sweep": "facade", "arch": arch.name, label: v, "tpot_ms": rep.tpot * 1e3, "hit_rate": rep.hit_rate,
             "cutoff": rep.cutoff_effective, "acceptance": rep.extras["acceptance_rate"],
             "hidden_prefetch_fraction": rep.extras["hidden_prefetch_fraction"],
             "prefetch_insertions": rep.counters["prefetch_insertions"]}
        print(json.dumps(r), flush=True)
        with open(a.out, "a") as f:
            f.write(json.dumps(r) + "\n")

    for v, rep in m.sweep("cutoff_layer", [0, 3, 6, 13, 20, 26], spec, hw, t, pol, **kw):
        row("cutoff_layer", v, rep)
    from dataclasses import replace

    pols = [replace(pol, policy=Policy(p), cutoff_layer=None if p != "draft_prefetch" else pol.cutoff_layer)
            for p in ("on_demand", "draft_prefetch", "gating_next_layer", "coarse_history")]
    for p, rep in zip(pols, m.compare_policies(spec, hw, t, pols, **kw)):
        row("policy", p.policy.value, rep)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["deepseek", "qwen", "mixtral", "mixtral_grid", "facade"])
    ap.add_argument("--out", default="profiles/sweeps_r1.jsonl")
    ap.add_argument("--steps", type=int, default=6)
    # the bit-exact CUDA-core K3 gives every policy point the same token
    # stream (its per-expert results do not depend on how experts are grouped
    # into launches); tcgen05 split choices do, which perturbs acceptance
    ap.add_argument("--ffn-impl", default="cuda_core")
    a = ap.parse_args()
    name = {"facade": "deepseek_v2_lite", "deepseek": "deepseek_v2_lite", "qwen": "qwen15_moe_a27b", "mixtral": "mixtral_8x7b",
            "mixtral_grid": "mixtral_8x7b"}[a.which]
    arch = get_arch(name)
    hw = HardwareSpec(gpu_memory=183_359 * 2**20, peak_non_expert_memory=24 * 10**9, pcie_bandwidth=55.5e9,
                      name="b200")
    t0 = time.time()
    # build the model once; engines share it
    seed_eng = SpecMoEEngine(arch, hw, b200_timings(arch, hw),
                             PolicySpec(policy=Policy.ON_DEMAND, prefetch_k=1, draft_length=2, acceptance_rate=1.0,
                                        seed=1234, cache_capacity_experts=arch.num_experts),
                             batch=1, max_tokens=64, cuda_graphs=False)
    state = seed_eng.model_state
    print(f"# model built in {time.time() - t0:.1f}s", file=sys.stderr, flush=True)
    pts = []
    if a.which == "facade":
        # the reference's own sweep / compare_policies entry points
        # (moesim simcore.py:518-564) over the real engine, one model build
        facade(arch, hw, state, a)
        seed_eng.close()
        return
    if a.which == "deepseek":
        pts.append(dict(policy="on_demand"))
        pts.append(dict())  # solver's cutoff (N-token window)
        pts.append(dict(window=False))  # verbatim reference budget
        for c in (0, 3, 6, 13, 20, 26):
            pts.append(dict(cutoff=c))
    elif a.which == "qwen":
        for N in (2, 4, 8):
            pts.append(dict(N=N))
        for B in (2, 4, 8):
            pts.append(dict(batch=B))
        for bud in (0.125, 0.5):
            pts.append(dict(budget=bud))
        pts.append(dict(policy="on_demand"))
    elif a.which == "mixtral_grid":
        # SURVEY 8(d) sweeps on config #2: budget (100 % = every expert
        # resident after warm-up, the HBM-bound verify), draft length, batch
        for bud in (0.125, 0.25, 0.5, 1.0):
            pts.append(dict(budget=bud))
        for N in (2, 8):
            pts.append(dict(N=N))
        for B in (2, 4):
            pts.append(dict(batch=B))
    else:
        for pol in ("on_demand", "draft_prefetch", "gating_next_layer", "coarse_history"):
            pts.append(dict(policy=pol))
        for c in (0, 4, 8):
            pts.append(dict(cutoff=c))
    with open(a.out, "a") as f:
        for kw in pts:
            r = point(arch, hw, state, steps=a.steps, ffn_impl=a.ffn_impl, **kw)
            r["sweep"] = a.which
            r["point"] = kw
            print(json.dumps(r), flush=True)
            f.write(json.dumps(r) + "\n")
    seed_eng.close()


if __name__ == "__main__":
    main()
