"""Measure the tcgen05 K3 launch for explicit (split_up, split_dn) choices.
python tools/tc_split_sweep.py"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2510_10302_b200 import kernels as K

def case(name, H, F, E, k, T, counts_fixed=None, iters=20):
    dev = "cuda"
    g = torch.Generator().manual_seed(0)
    x = torch.randn((T, H), generator=g).to(torch.bfloat16).to(dev)
    per = 3 * F * H * 2 * E
    R = max(1, int(np.ceil(600e6 / per)))
    pools = [torch.empty((E, 3 * F * H), dtype=torch.bfloat16, device=dev) for _ in range(R)]
    for i, p in enumerate(pools):
        K.fill_normal_(p, 100 + i, 0, 0.02)
    rng = np.random.default_rng(1)
    idx = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)
    off, perm, inv = K.moe_permute(torch.from_numpy(idx).to(dev), E)
    counts = np.bincount(idx.ravel(), minlength=E)
    U = int((counts > 0).sum())
    xp = torch.empty((T * k, H), dtype=torch.bfloat16, device=dev)
    h = torch.empty((T * k, F), dtype=torch.bfloat16, device=dev)
    y = torch.empty((T * k, H), dtype=torch.float32, device=dev)
    ws = torch.empty((K.tc_workspace_floats(T * k, H, F, 16, 16),), dtype=torch.float32, device=dev)
    plan = K.tc_plan(counts[counts > 0], H, F)
    res = {}
    for su, sd in [(1, 1), (1, 2), (1, 4), (1, 8), (2, 8), (4, 8), (1, 16), (8, 8), plan]:
        if su > H // 64 // 4 or sd > F // 64 // 4:
            continue
        for i in range(3):
            K.expert_ffn_tc(pools[i % R], list(range(E)), (1 << E) - 1, x, F, k, off, perm, xp, h, y, ws, su, sd)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        for i in range(iters):
            evs[i][0].record()
            K.expert_ffn_tc(pools[i % R], list(range(E)), (1 << E) - 1, x, F, k, off, perm, xp, h, y, ws, su, sd)
            evs[i][1].record()
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
        res[f"{su},{sd}"] = round(U * 3 * F * H * 2 / (ms / 1e3) / 1e9)
    print(json.dumps({"case": name, "U": U, "plan": plan, "GBps": res}), flush=True)

case("mixtral_T5", 4096, 14336, 8, 2, 5)
case("mixtral_T1_2exp", 4096, 14336, 8, 2, 1)
case("mixtral_1exp", 4096, 14336, 1, 1, 2)
case("mixtral_T72", 4096, 14336, 8, 2, 72)
case("deepseek_T5", 2048, 1408, 64, 6, 5)
case("qwen_T5", 2048, 1408, 60, 4, 5)
case("qwen_T72", 2048, 1408, 60, 4, 72)
case("deepseek_1exp", 2048, 1408, 1, 1, 2)
