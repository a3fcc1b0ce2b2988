"""Why is a late expert's K3 slower in the SD loop than back to back?
Time the tcgen05 K3 (1 Mixtral expert, 2 tokens) after: busy GPU; 4 ms host
idle; 4 ms idle + cross-stream event wait; 4 ms idle + a small same-stream
kernel first; 4 ms idle + a 64 MB memory-touching kernel first; 4 ms idle
with a 'keep-warm' spin kernel on a side stream during the gap."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2510_10302_b200 import kernels as K


def main(iters=12):
    H, F, T = 4096, 14336, 2
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
    su, sd = K.tc_plan_static(H, F)
    ws = torch.empty((max(1, K.tc_workspace_floats(T, H, F, su, sd)),), dtype=torch.float32, device=dev)
    side = torch.cuda.Stream()
    small = torch.zeros((1024,), device=dev)
    big = torch.zeros((16 << 20,), device=dev)  # 64 MB
    res = {}
    big2 = torch.zeros((29 << 20,), device=dev)  # 116 MB, like a decoded W2 segment
    hsrc = torch.empty((244 << 20,), dtype=torch.uint8).pin_memory()
    hdst = torch.empty((244 << 20,), dtype=torch.uint8, device=dev)
    cp = torch.cuda.Stream()
    small_dst = torch.empty((8 << 20,), dtype=torch.uint8, device=dev)
    for mode in ("prequeued_h2d_l2ring", "prequeued_w2", "prequeued_h2d", "prequeued_w2_h2d", "busy", "prequeued", "prequeued_big", "idle", "idle_event", "idle_small_first", "idle_big_first",
                 "idle_spin_side"):
        ts = []
        for i in range(iters + 2):
            if mode == "busy":
                torch.cuda._sleep(20000)
            elif mode.startswith("prequeued"):
                # launches queued ahead of the GPU behind a cross-stream event,
                # like a late expert waiting for its copy + decode
                torch.cuda.synchronize()
                with torch.cuda.stream(side):
                    torch.cuda._sleep(8_000_000)
                    if mode == "prequeued_big":
                        big.add_(1)
                    if mode in ("prequeued_w2", "prequeued_w2_h2d"):
                        big2.add_(1)
                    ev = torch.cuda.Event()
                    ev.record(side)
                if mode in ("prequeued_h2d", "prequeued_w2_h2d"):
                    # the next expert's copy is in flight on the copy engine
                    cp.wait_event(ev)
                    with torch.cuda.stream(cp):
                        hdst.copy_(hsrc, non_blocking=True)
                if mode == "prequeued_h2d_l2ring":
                    # same bytes, landing in one 8 MB (L2-resident) buffer
                    cp.wait_event(ev)
                    with torch.cuda.stream(cp):
                        for c in range(30):
                            small_dst.copy_(hsrc[c << 23:(c + 1) << 23], non_blocking=True)
                torch.cuda.current_stream().wait_event(ev)
            else:
                torch.cuda.synchronize()
                if mode == "idle_spin_side":
                    with torch.cuda.stream(side):
                        torch.cuda._sleep(8_000_000)  # ~4 ms of SM spinning, no memory traffic
                time.sleep(0.004)
                if mode == "idle_event":
                    with torch.cuda.stream(side):
                        small.add_(1)
                        ev = torch.cuda.Event()
                        ev.record(side)
                    torch.cuda.current_stream().wait_event(ev)
                elif mode == "idle_small_first":
                    small.add_(1)
                elif mode == "idle_big_first":
                    big.add_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            K.expert_ffn_tc(pool, [i % S], 1, x, F, 1, off, perm, xp, h, y, ws, su, sd)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        res[mode] = round(float(np.median([a.elapsed_time(b) for a, b in ts[2:]])) * 1e3, 1)
        print(json.dumps({mode: res[mode]}), flush=True)
    return res


if __name__ == "__main__":
    main()
