"""Acceptance diagnostics: graphs on/off, depth/width scaling."""
import json, sys
from dataclasses import replace
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec, ProfiledTimings
from paper_2510_10302_b200.engine import SpecMoEEngine
from paper_2510_10302_b200.model import get_arch

def run(name, graphs, steps=8, **ov):
    a = replace(get_arch(name), **ov)
    E = a.num_layers * a.num_experts
    hw = HardwareSpec(183_000_000_000, 24_000_000_000, 55e9)
    t = ProfiledTimings(1e-3, 1e-4, a.expert_bytes / 55e9)
    pol = PolicySpec(policy=Policy.ON_DEMAND, prefetch_k=1, draft_length=4, acceptance_rate=1.0, seed=1234,
                     cache_capacity_experts=max(a.num_experts, min(E, 32)))
    eng = SpecMoEEngine(a, hw, t, pol, batch=1, host_distinct=min(E, 32), max_tokens=256, cuda_graphs=graphs)
    g = torch.Generator().manual_seed(1000)
    eng.prefill(torch.randint(0, a.vocab, (1, 32), generator=g))
    for _ in range(steps):
        eng.step()
    rep = eng.report()
    toks = eng.seqs[0][32:]
    print(json.dumps({"arch": name, "graphs": graphs, **ov, "acc": round(rep.extras["acceptance_rate"], 3),
                      "tokens": toks[:16]}), flush=True)
    eng.close()
    torch.cuda.empty_cache()

run("tiny", True, expert_spread=0.1)
run("tiny", False, expert_spread=0.1)
run("mixtral_8x7b", False, expert_spread=0.05, embed_std=1.0)
for L in (1, 2, 4):
    run("mixtral_8x7b", True, num_layers=L, expert_spread=0.05)
run("mixtral_8x7b", True, num_layers=4, hidden=1024, num_heads=8, num_kv_heads=2, ffn=3584, expert_spread=0.05)
run("mixtral_8x7b", True, num_layers=4, vocab=512, expert_spread=0.05)
