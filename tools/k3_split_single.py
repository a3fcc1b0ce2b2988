"""Split-K plans for ONE late expert (Mixtral, T routed tokens) on the
tcgen05 K3: time every (split_up, split_dn) pair back to back and with a
concurrent 244 MB H2D copy in flight (the SD loop's situation).
python tools/k3_split_single.py [T]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2510_10302_b200 import kernels as K


def main(T=2, iters=10):
    H, F = 4096, 14336
    dev = "cuda"
    S = 8
    pool = torch.empty((S, 3 * F * H), dtype=torch.bfloat16, device=dev)
    K.fill_normal_(pool, 7, 0, 0.02)
    x = torch.randn((T, H), device=dev).to(torch.bfloat16)
    idx = torch.zeros((T, 1), dtype=torch.int32, device=dev)
    off, perm, inv = K.moe_permute(idx, 1)
    h = torch.empty((T, F), dtype=torch.bfloat16, device=dev)
    y = torch.empty((T, H), dtype=torch.float32, device=dev)
    xp = torch.empty((T, H), dtype=torch.bfloat16, device=dev)
    ws = torch.empty((K.tc_workspace_floats(T, H, F, 16, 16),), dtype=torch.float32, device=dev)
    hsrc = torch.empty((244 << 20,), dtype=torch.uint8).pin_memory()
    hdst = torch.empty((244 << 20,), dtype=torch.uint8, device=dev)
    cp = torch.cuda.Stream()
    eb = 3 * F * H * 2
    out = []
    for su in (1, 2, 3, 4, 5, 9):
        for sd in (2, 4, 5, 9, 14):
            row = {"T": T, "split_up": su, "split_dn": sd}
            for mode in ("alone", "h2d"):
                ts = []
                for i in range(iters + 2):
                    torch.cuda.synchronize()
                    if mode == "h2d":
                        with torch.cuda.stream(cp):
                            hdst.copy_(hsrc, non_blocking=True)
                        torch.cuda._sleep(200000)  # let the copy get going
                    else:
                        torch.cuda._sleep(20000)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    K.expert_ffn_tc(pool, [i % S], 1, x, F, 1, off, perm, xp, h, y, ws, su, sd)
                    b.record()
                    ts.append((a, b))
                torch.cuda.synchronize()
                us = float(np.median([a.elapsed_time(b) for a, b in ts[2:]])) * 1e3
                row[mode] = {"us": round(us, 1), "tbs": round(eb / us / 1e6, 3)}
            out.append(row)
            print(json.dumps(row), flush=True)
    return out


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
