#!/bin/bash
mkdir -p gpurun_out
python - <<'PY' 2>&1 | grep -E "arch|Error|Trace" | tail -20
import json, sys, time
from dataclasses import replace
sys.path.insert(0, ".")
import torch
from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec, ProfiledTimings
from paper_2510_10302_b200.engine import SpecMoEEngine
from paper_2510_10302_b200.model import get_arch
def run(name, steps=16, **ov):
    a = replace(get_arch(name), **ov)
    E = a.num_layers * a.num_experts
    hw = HardwareSpec(183_000_000_000, 24_000_000_000, 55e9)
    t = ProfiledTimings(1e-3, 1e-4, a.expert_bytes / 55e9)
    pol = PolicySpec(policy=Policy.ON_DEMAND, prefetch_k=1, draft_length=4, acceptance_rate=1.0, seed=1234,
                     cache_capacity_experts=E)
    t0 = time.time()
    eng = SpecMoEEngine(a, hw, t, pol, batch=1, max_tokens=200)
    g = torch.Generator().manual_seed(1000)
    eng.prefill(torch.randint(0, a.vocab, (1, 64), generator=g))
    for _ in range(steps):
        eng.step()
    rep = eng.report()
    print(json.dumps({"arch": name, **ov, "acc": round(rep.extras["acceptance_rate"], 3),
                      "emit": round(rep.emitted_tokens / len(rep.iterations), 2), "s": round(time.time() - t0)}), flush=True)
    eng.close(); del eng; torch.cuda.empty_cache()
for sp in (0.01, 0.02, 0.03):
    run("mixtral_8x7b", expert_spread=sp)
for sp in (0.02, 0.04):
    run("deepseek_v2_lite", expert_spread=sp)
    run("qwen15_moe_a27b", expert_spread=sp)
PY
