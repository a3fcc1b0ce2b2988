"""HBM copy bandwidth of an SM kernel alone vs while the copy engine streams
a pinned host buffer into HBM (the SD loop's situation): the in-situ HBM
peak against which a verify-time kernel can be judged.  Prints GB/s of
read+write for a 2 GiB -> 2 GiB elementwise copy (torch mul by 1, an SM
kernel), and for a pure read stream (a 2 GiB reduction), median of 10."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch


def main(iters=10):
    dev = "cuda"
    n = 1 << 30  # bf16 elements: 2 GiB
    a = torch.ones((n,), dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    hsrc = torch.empty((1 << 30,), dtype=torch.uint8).pin_memory()
    hdst = torch.empty((1 << 30,), dtype=torch.uint8, device=dev)
    cp = torch.cuda.Stream()
    res = {}
    red = torch.empty((1,), dtype=torch.float32, device=dev)
    for mode in ("alone", "with_h2d", "read_alone", "read_with_h2d"):
        ts = []
        for i in range(iters + 2):
            torch.cuda.synchronize()
            if mode.endswith("with_h2d"):
                with torch.cuda.stream(cp):
                    hdst.copy_(hsrc, non_blocking=True)  # ~19 ms at the link peak
                torch.cuda._sleep(100000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if mode.startswith("read"):
                torch.sum(a.view(1, -1), dim=(1,), dtype=torch.float32, out=red)  # pure read stream
            else:
                torch.mul(a, 1, out=b)
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        ms = float(np.median([x.elapsed_time(y) for x, y in ts[2:]]))
        byts = 2 * n * (1 if mode.startswith("read") else 2)
        res[mode] = {"ms": round(ms, 3), "gbs": round(byts / (ms / 1e3) / 1e9, 1)}
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    main()
