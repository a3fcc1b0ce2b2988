"""Microbenchmark of the verify-MoE kernels at BASELINE shapes (resident pool).

Reports, per config, the K3 (expert_ffn up+down) time and achieved HBM GB/s
of algorithmic bytes (distinct routed experts x expert bytes + activations),
plus K1 router latency.  Usage: python tools/bench_kernels.py [--json out]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2510_10302_b200 import kernels as K  # noqa: E402

CASES = {
    "mixtral_T5": dict(H=4096, F=14336, E=8, k=2, T=5),
    "mixtral_T1": dict(H=4096, F=14336, E=8, k=2, T=1),
    "mixtral_T9": dict(H=4096, F=14336, E=8, k=2, T=9),
    "mixtral_T72": dict(H=4096, F=14336, E=8, k=2, T=72),
    # prefill-sized batches: 128 / 512 routed tokens per expert (the
    # tensor-core regime: report tensor-pipe use for B(N+1) >= 32)
    "mixtral_T512": dict(H=4096, F=14336, E=8, k=2, T=512),
    "mixtral_T2048": dict(H=4096, F=14336, E=8, k=2, T=2048),
    "deepseek_T5": dict(H=2048, F=1408, E=64, k=6, T=5),
    "qwen_T5": dict(H=2048, F=1408, E=60, k=4, T=5),
    "qwen_T72": dict(H=2048, F=1408, E=60, k=4, T=72),
    "mixtral_1exp": dict(H=4096, F=14336, E=1, k=1, T=2),
}


def run_case(name, H, F, E, k, T, iters=20, warmup=5):
    dev = "cuda"
    g = torch.Generator().manual_seed(0)
    x = (torch.randn((T, H), generator=g)).to(torch.bfloat16).to(dev)
    # enough distinct copies of the expert set that consecutive iterations
    # never hit L2 (126 MB): rotate among R pools
    per = 3 * F * H * 2 * E
    R = max(1, int(np.ceil(600e6 / per)))
    pools = [torch.empty((E, 3 * F * H), dtype=torch.bfloat16, device=dev) for _ in range(R)]
    for i, p in enumerate(pools):
        K.fill_normal_(p, 100 + i, 0, 0.02)
    rw = (torch.randn((E, H), generator=g) / H**0.5).to(torch.bfloat16).to(dev)
    w, idx, _, _ = K.router_topk(x, rw, k, True)
    off, perm, inv = K.moe_permute(idx, E)
    ids = idx.cpu().numpy().ravel()
    U = len(set(ids.tolist()))
    maxtok = int(np.bincount(ids, minlength=E).max())
    h = torch.empty((T * k, F), dtype=torch.bfloat16, device=dev)
    y = torch.empty((T * k, H), dtype=torch.float32, device=dev)
    slots = list(range(E))
    mask = (1 << E) - 1
    st = torch.cuda.current_stream()

    xp = torch.empty((T * k, H), dtype=torch.bfloat16, device=dev)
    su, sd = K.tc_plan(np.bincount(ids, minlength=E), H, F)
    ws = torch.empty((max(1, K.tc_workspace_floats(T * k, H, F, su, sd)),), dtype=torch.float32, device=dev)

    sync = torch.zeros((1,), dtype=torch.int32, device=dev)

    def once(i, phase="both"):
        if phase == "tcf":
            K.expert_ffn_tc_fused(pools[i % R], slots, mask, x, F, k, off, perm, xp, h, y, ws, sd, sync)
            return
        if phase == "tc":
            K.expert_ffn_tc(pools[i % R], slots, mask, x, F, k, off, perm, xp, h, y, ws, su, sd)
            return
        K.expert_ffn(pools[i % R], slots, mask, x, F, k, off, perm, h, y, maxtok, phase=phase)

    for i in range(warmup):
        once(i)
    res = {}
    for phase in ("both", "up", "down", "tc", "tcf"):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        torch.cuda.synchronize()
        for i in range(iters):
            evs[i][0].record(st)
            once(i, phase)
            evs[i][1].record(st)
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
        wbytes = {"both": 3, "up": 2, "down": 1, "tc": 3, "tcf": 3}[phase] * F * H * 2 * U
        act = T * k * (H * 2 + F * 2 * 2 + H * 4)
        res[phase] = {"ms": ms, "GBps": (wbytes + act) / (ms / 1e3) / 1e9, "weight_bytes": wbytes}
    # router latency
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for i in range(iters):
        evs[i][0].record(st)
        K.router_topk(x, rw, k, True)
        evs[i][1].record(st)
    torch.cuda.synchronize()
    res["router_us"] = float(np.median([a.elapsed_time(b) for a, b in evs])) * 1e3
    res.update(dict(name=name, H=H, F=F, E=E, k=k, T=T, distinct_experts=U, max_tokens_per_expert=maxtok))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    out = []
    for name in a.cases.split(","):
        r = run_case(name, iters=a.iters, warmup=a.warmup, **CASES[name])
        out.append(r)
        print(json.dumps(r))
    if a.json:
        Path(a.json).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
