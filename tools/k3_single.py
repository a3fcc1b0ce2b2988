"""K3 for ONE late expert (the bench's regime: each demand-loaded expert runs
alone after its copy lands), Mixtral shapes, 1..4 routed tokens (optionally with a concurrent 244 MB H2D copy per launch).  Times the
tcgen05 launcher (static split plan), the fused tcgen05 kernel and the
CUDA-core kernel with CUDA events, rotating over 8 slots (>= 2.8 GB, no L2
reuse), each launch preceded by an idle gap (like a stream waiting on a
copy event).  Usage: python tools/k3_single.py [iters gap Ts impls [h2d]]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2510_10302_b200 import kernels as K


def main(iters=20, gap_cycles=20000, Ts=(1, 2, 3, 4), impls=("tc", "tc_fused", "cuda_core"), h2d=False):
    H, F = 4096, 14336
    dev = "cuda"
    S = 8
    pool = torch.empty((S, 3 * F * H), dtype=torch.bfloat16, device=dev)
    K.fill_normal_(pool, 7, 0, 0.02)
    eb = 3 * F * H * 2
    sync = torch.zeros((1,), dtype=torch.int32, device=dev)
    side = torch.cuda.Stream()
    side_buf = torch.zeros((1024,), device=dev)
    if h2d:  # a concurrent host->HBM copy in flight during every launch (the SD loop's situation)
        hsrc = torch.empty((244 << 20,), dtype=torch.uint8).pin_memory()
        hdst = torch.empty((244 << 20,), dtype=torch.uint8, device=dev)
    from paper_2510_10302_b200 import _native

    lib = _native.load()
    spans = torch.zeros((iters + 3, 2), dtype=torch.int64, device=dev)
    out = []
    for T in Ts:
        g = torch.Generator().manual_seed(T)
        x = torch.randn((T, H), generator=g).to(torch.bfloat16).to(dev)
        idx = torch.zeros((T, 1), dtype=torch.int32, device=dev)
        off, perm, inv = K.moe_permute(idx, 1)
        h = torch.empty((T, F), dtype=torch.bfloat16, device=dev)
        y = torch.empty((T, H), dtype=torch.float32, device=dev)
        xp = torch.empty((T, H), dtype=torch.bfloat16, device=dev)
        su, sd = K.tc_plan_static(H, F)
        ws = torch.empty((max(1, K.tc_workspace_floats(T, H, F, su, sd)),), dtype=torch.float32, device=dev)
        wsu = torch.zeros((K.tc_units_workspace_floats(T, H, F),), dtype=torch.float32, device=dev)
        act = T * (H * 2 + 2 * F * 2 + H * 4)
        row = {"T": T, "split": [su, sd], "gap_cycles": gap_cycles, "h2d": h2d}
        for name in impls:
            ms = []
            for i in range(iters + 3):
                slot = i % S
                if gap_cycles < 0:
                    # truly idle GPU for |gap| microseconds (empty streams), then
                    # the launch waits on an event of another stream, as the
                    # bench's late experts wait on their decode
                    torch.cuda.synchronize()
                    time.sleep(-gap_cycles / 1e6)
                    with torch.cuda.stream(side):
                        side_buf.add_(1)
                        ev = torch.cuda.Event()
                        ev.record(side)
                    torch.cuda.current_stream().wait_event(ev)
                else:
                    if h2d:
                        torch.cuda.synchronize()
                        with torch.cuda.stream(side):
                            hdst.copy_(hsrc, non_blocking=True)
                    torch.cuda._sleep(gap_cycles)  # busy gap
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                lib.spmoe_k3_devtiming(spans[i].data_ptr())
                a.record()
                if name == "tc":
                    K.expert_ffn_tc(pool, [slot], 1, x, F, 1, off, perm, xp, h, y, ws, su, sd)
                elif name == "tc_units":
                    K.expert_ffn_tc_units(pool, [slot], 1, x, F, 1, off, perm, T, xp, None, y, wsu)
                elif name == "tc_fused":
                    K.expert_ffn_tc_fused(pool, [slot], 1, x, F, 1, off, perm, xp, h, y, ws, sd, sync)
                else:
                    K.expert_ffn(pool, [slot], 1, x, F, 1, off, perm, h, y, T)
                b.record()
                ms.append((a, b))
            torch.cuda.synchronize()
            lib.spmoe_k3_devtiming(None)
            t = [a.elapsed_time(b) for a, b in ms[3:]]
            med = float(np.median(t))
            row[name] = {"us": round(med * 1e3, 1), "tbs": round((eb + act) / (med / 1e3) / 1e12, 3)}
            sp = spans.cpu().numpy()[3:]
            if (sp[:, 0] > 0).all():
                dmed = float(np.median(sp[:, 1] - sp[:, 0])) / 1e3
                row[name]["device_us"] = round(dmed, 1)
                row[name]["device_tbs"] = round((eb + act) / (dmed / 1e6) / 1e12, 3)
            spans.zero_()
        out.append(row)
        print(json.dumps(row), flush=True)
    return out


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if len(a) > 0 else 20, int(a[1]) if len(a) > 1 else 20000,
         tuple(int(t) for t in a[2].split(",")) if len(a) > 2 else (1, 2, 3, 4),
         tuple(a[3].split(",")) if len(a) > 3 else ("tc", "tc_fused", "cuda_core"),
         len(a) > 4 and a[4] == "h2d")
