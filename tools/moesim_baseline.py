"""the reference simulator's own wall time on the same
configs, measured HERE (the build container: `/root/reference` does not
exist on the GPU box, so this baseline cannot run there).

For each bench preset (Mixtral-8x7B / DeepSeek-V2-Lite / Qwen1.5-MoE at a
25 % budget, the tiny config #1) the same ModelSpec / HardwareSpec (the
B200's measured pinned H2D peak) / ProfiledTimings (calibrate.b200_timings)
/ PolicySpec the bench uses are written with this package's write_config
and loaded with moesim.load_config; moesim.generate_synthetic_trace draws
the activation trace (100 output tokens, seed 1234) and moesim.simulate
runs it single-threaded, best of 3.  The shipped pkg/configs run as well.
Reported: wall ms per run and per simulated token, the simulator's own
TPOT.  A reported baseline (the reference's CPU path is a simulator; it
moves no bytes), not a target.

  PYTHONPATH=/root/reference/pkg/src python tools/moesim_baseline.py [OUT.json]
"""
from __future__ import annotations

import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import moesim  # noqa: E402
from moesim.trace import generate_synthetic_trace  # noqa: E402

from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec  # noqa: E402
from paper_2510_10302_b200.calibrate import b200_timings  # noqa: E402
from paper_2510_10302_b200.config import write_config  # noqa: E402
from paper_2510_10302_b200.model import get_arch, model_spec_for  # noqa: E402

PRESETS = {  # bench.py CONFIGS
    "mixtral": dict(arch="mixtral_8x7b", budget=0.25, N=4),
    "deepseek": dict(arch="deepseek_v2_lite", budget=0.25, N=4),
    "qwen": dict(arch="qwen15_moe_a27b", budget=0.25, N=4),
    "tiny": dict(arch="tiny", budget=0.375, N=4),
}
TOKENS = 100
H2D_GBS = 55.6  # the gpurun boxes' measured pinned H2D peak (bench lines, profiles/r2)
ACCEPT = 0.85  # acceptance measured by the bench at the Mixtral config


def timed(fn, reps=3):
    best, out = None, None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


def run_specs(model, hw, timings, policy):
    trace = generate_synthetic_trace(model, TOKENS, seed=policy.seed)
    wall, rep = timed(lambda: moesim.simulate(model, hw, timings, policy, trace))
    return {"wall_ms": round(wall * 1e3, 2), "wall_ms_per_token": round(wall * 1e3 / TOKENS, 3),
            "simulated_tpot_ms": round(rep.tpot * 1e3, 3), "simulated_hit_rate": round(rep.hit_rate, 4)}


def main(out=None):
    res = {"threads": 1, "cpu_count": os.cpu_count(), "tokens": TOKENS, "configs": {}}
    with tempfile.TemporaryDirectory() as td:
        for name, c in PRESETS.items():
            arch = get_arch(c["arch"])
            model = model_spec_for(arch)
            hw = HardwareSpec(gpu_memory=183_359 * 2**20, peak_non_expert_memory=24 * 10**9,
                              pcie_bandwidth=H2D_GBS * 1e9, name="b200")
            timings = b200_timings(arch, hw)
            cap = max(arch.num_experts, int(round(c["budget"] * arch.num_layers * arch.num_experts)))
            policy = PolicySpec(policy=Policy("draft_prefetch"), prefetch_k=1 if arch.num_experts <= 16 else arch.top_k,
                                draft_length=c["N"], acceptance_rate=ACCEPT, seed=1234, cache_capacity_experts=cap)
            path = Path(td) / f"{name}.yaml"
            write_config(path, model, hw, timings, policy)
            specs = moesim.load_config(path)  # the reference's own parser
            res["configs"][name] = run_specs(*specs)
            print(name, res["configs"][name], flush=True)
    for y in sorted(Path("/root/reference/pkg/configs").glob("*.yaml")):
        res["configs"]["pkg/" + y.stem] = r = run_specs(*moesim.load_config(y))
        print(y.stem, r, flush=True)
    if out:
        Path(out).write_text(json.dumps(res, indent=1))
    return res


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
