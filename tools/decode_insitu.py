"""Why is an XC segment decode slower inside the runtime (≈ 77 µs) than back
to back (≈ 46 µs)?  Times one segment decode (Mixtral-8x7B W1, one launch)
under: the same buffers back to back; rotating output slots and input blobs
(cold TLB / L2); an idle gap before each launch; a concurrent H2D copy; and
the runtime's situation (idle gap + rotating buffers + H2D).  Reports the
median launch time by CUDA events and by device clock (globaltimer span of
the launch), and the device-clock algorithmic GB/s (segment bytes in + raw
bytes out) and fraction of the measured HBM copy peak.
python tools/decode_insitu.py"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2510_10302_b200 import _native
from paper_2510_10302_b200 import codec as X
from paper_2510_10302_b200.model import fill_expert_blob, get_arch


def main(iters=12):
    a = get_arch("mixtral_8x7b")
    dev = torch.device("cuda", 0)
    src = torch.empty((a.expert_elems,), dtype=torch.bfloat16, device=dev)
    enc = X.XcEncoder(X.expert_segments(a.ffn, a.hidden), dev)
    blobs, hdrs = [], []
    for r in range(3):
        fill_expert_blob(src, a, 1234, r)
        h = enc.plan(src)
        blobs.append(enc.encode(src, h).clone())
        hdrs.append(h)
    slots = torch.empty((8, a.expert_elems), dtype=torch.bfloat16, device=dev)
    lib = _native.load()
    st = torch.cuda.current_stream()
    hsrc = torch.empty((244 << 20,), dtype=torch.uint8).pin_memory()
    hdst = torch.empty((244 << 20,), dtype=torch.uint8, device=dev)
    cp = torch.cuda.Stream()
    spans = torch.zeros((iters + 2, 2), dtype=torch.int64, device=dev)
    g0 = hdrs[0].seg
    alg = int(g0[1].off_lut) + 2 * int(g0[0].n)  # segment 0 incl. header: bytes in + out
    try:
        peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        peak = 6556.2
    res = {}
    for mode in ("same_b2b", "rotate_b2b", "same_idle", "rotate_idle", "same_h2d", "rotate_idle_h2d"):
        ts = []
        for i in range(iters + 2):
            rot = mode.startswith("rotate")
            b, h = (blobs[i % 3], hdrs[i % 3]) if rot else (blobs[0], hdrs[0])
            out = slots[i % 8] if rot else slots[0]
            if "idle" in mode or "h2d" in mode:
                torch.cuda.synchronize()
                if "h2d" in mode:
                    with torch.cuda.stream(cp):
                        hdst.copy_(hsrc, non_blocking=True)
                if "idle" in mode:
                    time.sleep(0.001)
                else:
                    torch.cuda._sleep(200000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            spans[i].zero_()
            _native.check("spmoe_xc_decode_segments_timed", lib.spmoe_xc_decode_segments_timed(
                C.c_void_p(b.data_ptr()), C.addressof(h), 0, 1, C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream),
                C.c_void_p(spans[i].data_ptr())))
            e1.record(st)
            ts.append((e0, e1))
        torch.cuda.synchronize()
        us = float(np.median([x.elapsed_time(y) for x, y in ts[2:]])) * 1e3
        sp = spans.cpu().numpy()[2:]
        dus = float(np.median(sp[:, 1] - sp[:, 0])) / 1e3
        res[mode] = {"events_us": round(us, 1), "device_us": round(dus, 1),
                     "device_gbs": round(alg / dus / 1e3, 1), "frac": round(alg / dus / 1e3 / peak, 3)}
        print(json.dumps({mode: res[mode]}), flush=True)
    return res


if __name__ == "__main__":
    main()
