"""Acceptance rate of the synthetic draft/target pair vs init knobs.
python tools/tune_acceptance.py ARCH '[{"expert_spread":0.1,"embed_std":1.0}, ...]' [steps]"""
import json, sys, time
from dataclasses import replace
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec, ProfiledTimings
from paper_2510_10302_b200.engine import SpecMoEEngine
from paper_2510_10302_b200.model import get_arch

name = sys.argv[1]
variants = json.loads(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
for ov in variants:
    a = replace(get_arch(name), **ov)
    E = a.num_layers * a.num_experts
    hw = HardwareSpec(183_000_000_000, 24_000_000_000, 55e9)
    t = ProfiledTimings(1e-3, 1e-4, a.expert_bytes / 55e9)
    pol = PolicySpec(policy=Policy.ON_DEMAND, prefetch_k=1, draft_length=4, acceptance_rate=1.0, seed=1234,
                     cache_capacity_experts=max(a.num_experts, min(E, 32)))
    t0 = time.time()
    eng = SpecMoEEngine(a, hw, t, pol, batch=1, host_distinct=min(E, 32), max_tokens=256)
    g = torch.Generator().manual_seed(1000)
    eng.prefill(torch.randint(0, a.vocab, (1, 64), generator=g))
    for _ in range(steps):
        eng.step()
    rep = eng.report()
    print(json.dumps({"arch": name, **ov, "acceptance": round(rep.extras["acceptance_rate"], 3),
                      "emitted_per_iter": round(rep.emitted_tokens / len(rep.iterations), 3),
                      "setup_s": round(time.time() - t0, 1)}), flush=True)
    eng.close()
    del eng
    torch.cuda.empty_cache()
