"""Round-2 diagnostics: (1) EP vs local verify-MoE intermediates on the tiny
config; (2) Mixtral acceptance under the K3 variants (static split plan,
per-launch plan, CUDA-core)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch

from paper_2510_10302_b200 import kernels as K
from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec
from paper_2510_10302_b200.calibrate import b200_timings
from paper_2510_10302_b200.engine import SpecMoEEngine
from paper_2510_10302_b200.model import get_arch


def ep_debug():
    from test_engine_gpu import make_engine, prompts, bits

    stash = {}
    orig = SpecMoEEngine._shared_and_combine

    def spy(self, l, xn, resid, s, w, idx, sg, y, inv, slots):
        T = xn.shape[0]
        stash.setdefault(("ep" if self.ep is not None else "loc", l), (y[: T * self.arch.top_k].clone(), xn.clone()))
        return orig(self, l, xn, resid, s, w, idx, sg, y, inv, slots)

    SpecMoEEngine._shared_and_combine = spy
    kw = dict(policy_kind="on_demand", cutoff=None, capacity=12, batch=1, capture=(0,))
    for ep in (True, False):
        eng = make_engine(expert_parallel=ep, **kw)
        eng.prefill(prompts(1))
        eng.step()
        torch.cuda.synchronize()
        eng.close()
    SpecMoEEngine._shared_and_combine = orig
    for l in range(4):
        a, b = stash.get(("ep", l)), stash.get(("loc", l))
        if a is None or b is None:
            continue
        ya, yb = a[0].cpu().numpy(), b[0].cpu().numpy()
        xa, xb = bits(a[1]), bits(b[1])
        rows = [i for i in range(ya.shape[0]) if not np.array_equal(ya[i].view(np.uint32), yb[i].view(np.uint32))]
        print(json.dumps({"layer": l, "x_equal": bool(np.array_equal(xa, xb)), "y_rows": ya.shape[0],
                          "y_rows_differ": rows, "max_abs": float(np.abs(ya - yb).max())}), flush=True)


def accept_variants(steps=8):
    arch = get_arch("mixtral_8x7b")
    E_all = arch.num_layers * arch.num_experts
    hw = HardwareSpec(gpu_memory=183_359 * 2**20, peak_non_expert_memory=24 * 10**9, pcie_bandwidth=55.5e9, name="b200")
    timings = b200_timings(arch, hw)
    pol = PolicySpec(policy=Policy.DRAFT_PREFETCH, prefetch_k=1, draft_length=4, acceptance_rate=1.0, seed=1234,
                     cache_capacity_experts=64)
    state = None
    keep = []
    for name, impl, dyn in (("static", "auto", False), ("cuda_core", "cuda_core", False), ("dynamic", "auto", True)):
        if dyn:
            # old per-launch plan: split chosen from the launch's own counts
            def _ffn(self, pool, slots, mask, xn, F, k, offsets, perm, h, y, maxtok, s, counts=None):
                if self._use_tc(F, maxtok):
                    rows = xn.shape[0] * k
                    su, sd = K.tc_plan(counts if counts is not None else [maxtok], self.arch.hidden, F, self.num_sms)
                    K.expert_ffn_tc(pool, slots, mask, xn, F, k, offsets, perm, s.xp[:rows], h, y, s.ysplit, su, sd)
                else:
                    K.expert_ffn(pool, slots, mask, xn, F, k, offsets, perm, h, y, maxtok)
            SpecMoEEngine._ffn = _ffn
        eng = SpecMoEEngine(arch, hw, timings, pol, batch=1, max_tokens=64 + 64 * 5, window_tokens=4,
                            ffn_impl=impl, model_state=state)
        state = eng.model_state
        g = torch.Generator().manual_seed(1000)
        eng.prefill(torch.randint(0, arch.vocab, (1, 64), generator=g))
        em = [sum(eng.step()) for _ in range(steps)]
        rep = eng.report()
        print(json.dumps({"variant": name, "acc": rep.extras["acceptance_rate"], "emitted": em,
                          "tokens": eng.seqs[0][64:96]}), flush=True)
        keep.append(eng)
    for eng in reversed(keep):
        eng.close()


def spread_sweep(steps=20):
    """Acceptance of the synthetic Mixtral pair vs expert_spread (values
    only: bytes and FLOPs are identical), bench prompt and policy."""
    from dataclasses import replace

    for spread in (0.005, 0.003, 0.002, 0.001):
        arch = replace(get_arch("mixtral_8x7b"), expert_spread=spread)
        hw = HardwareSpec(gpu_memory=183_359 * 2**20, peak_non_expert_memory=24 * 10**9, pcie_bandwidth=55.5e9,
                          name="b200")
        pol = PolicySpec(policy=Policy.DRAFT_PREFETCH, prefetch_k=1, draft_length=4, acceptance_rate=1.0,
                         seed=1234, cache_capacity_experts=64)
        eng = SpecMoEEngine(arch, hw, b200_timings(arch, hw), pol, batch=1, max_tokens=64 + 64 * 5, window_tokens=4)
        for seed in (1000, 1001):
            g = torch.Generator().manual_seed(seed)
            eng.prefill(torch.randint(0, arch.vocab, (1, 64), generator=g))
            em = [sum(eng.step()) for _ in range(steps)]
            print(json.dumps({"spread": spread, "prompt_seed": seed, "acc": eng.accepted_total / eng.drafted_total,
                              "emitted": em}), flush=True)
        eng.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    what = sys.argv[1:] or ["ep", "acc"]
    if "ep" in what:
        ep_debug()
    if "acc" in what:
        accept_variants()
    if "spread" in what:
        spread_sweep()
