"""Two-phase tcgen05 K3 (expert_ffn_tc) at prefill-sized token counts:
host-timed calls (synchronised) and CUDA-event timing, Mixtral shapes,
8 experts, T routed tokens (top-2).  python tools/tc_large_t.py [T ...]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2510_10302_b200 import kernels as K


def main(Ts):
    H, F, E, k = 4096, 14336, 8, 2
    dev = "cuda"
    pool = torch.empty((E, 3 * F * H), dtype=torch.bfloat16, device=dev)
    K.fill_normal_(pool, 5, 0, 0.02)
    g = torch.Generator().manual_seed(0)
    rw = (torch.randn((E, H), generator=g) / H**0.5).to(torch.bfloat16).to(dev)
    for T in Ts:
        x = torch.randn((T, H), generator=g).to(torch.bfloat16).to(dev)
        w, idx, _, _ = K.router_topk(x, rw, k, True)
        off, perm, inv = K.moe_permute(idx, E)
        ids = idx.cpu().numpy().ravel()
        counts = np.bincount(ids, minlength=E)
        su, sd = K.tc_plan(counts, H, F)
        xp = torch.empty((T * k, H), dtype=torch.bfloat16, device=dev)
        h = torch.empty((T * k, F), dtype=torch.bfloat16, device=dev)
        y = torch.empty((T * k, H), dtype=torch.float32, device=dev)
        ws = torch.empty((max(1, K.tc_workspace_floats(T * k, H, F, su, sd)),), dtype=torch.float32, device=dev)
        call = lambda: K.expert_ffn_tc(pool, list(range(E)), (1 << E) - 1, x, F, k, off, perm, xp, h, y, ws, su, sd)
        call()
        torch.cuda.synchronize()
        hs = []
        for _ in range(5):
            t0 = time.perf_counter()
            call()
            torch.cuda.synchronize()
            hs.append((time.perf_counter() - t0) * 1e3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            call()
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"T": T, "max_per_expert": int(counts.max()), "split": [su, sd],
                          "host_ms": round(float(np.median(hs)), 3), "event_ms": round(a.elapsed_time(b) / 5, 3)}),
              flush=True)


if __name__ == "__main__":
    main([int(t) for t in sys.argv[1:]] or [64, 128, 256, 512, 1024, 2048])
