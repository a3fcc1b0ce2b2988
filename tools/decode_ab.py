"""A/B of the XC segment decode across library builds on ONE box (box-to-box
spread is ~5 %): every build in argv (paths to libspmoe.so variants, plus
an A/B environment switch the build reads as "path:value" in SPMOE_XC_DEC) encodes the same Mixtral-8x7B
expert with its own encoder (builds may differ in format details that keep
the header layout) and decodes its W1 segment back to back, interleaved
round-robin, timed by device clock (globaltimer span of the launch).
python tools/decode_ab.py paper_2510_10302_b200/libspmoe.so _variants/x.so"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2510_10302_b200 import codec as X
from paper_2510_10302_b200.model import fill_expert_blob, get_arch


def main(paths, reps=30):
    a = get_arch("mixtral_8x7b")
    dev = torch.device("cuda", 0)
    src = torch.empty((a.expert_elems,), dtype=torch.bfloat16, device=dev)
    fill_expert_blob(src, a, 1234, 0)
    segs = np.asarray(X.expert_segments(a.ffn, a.hidden), dtype=np.int64)
    import shutil
    import tempfile

    libs = []
    tmpd = tempfile.mkdtemp()
    out = torch.empty((a.expert_elems,), dtype=torch.bfloat16, device=dev)
    spans = torch.zeros((len(paths), reps, 2), dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream()
    for i, spec in enumerate(paths):
        path, _, var = spec.partition(":")
        cp = os.path.join(tmpd, f"v{i}.so")  # a private copy: its own statics
        shutil.copy(path, cp)
        lib = C.CDLL(cp)
        fn = lib.spmoe_xc_decode_segments_timed
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p] * 2 + [C.c_int] * 2 + [C.c_void_p] * 3
        lib.spmoe_xc_work_bytes.restype = C.c_size_t
        lib.spmoe_xc_work_bytes.argtypes = [C.c_int, C.c_void_p]
        work = torch.empty((int(lib.spmoe_xc_work_bytes(len(segs), segs.ctypes.data)),), dtype=torch.uint8, device=dev)
        h = X.XcHeader()
        assert lib.spmoe_xc_plan(C.c_void_p(src.data_ptr()), C.c_int(len(segs)), C.c_void_p(segs.ctypes.data),
                                 C.c_void_p(work.data_ptr()), C.c_void_p(C.addressof(h)),
                                 C.c_void_p(st.cuda_stream)) == 0
        blob = torch.empty((int(h.blob_bytes),), dtype=torch.uint8, device=dev)
        assert lib.spmoe_xc_encode(C.c_void_p(src.data_ptr()), C.c_void_p(C.addressof(h)),
                                   C.c_void_p(work.data_ptr()), C.c_void_p(blob.data_ptr()),
                                   C.c_void_p(st.cuda_stream)) == 0
        os.environ["SPMOE_XC_DEC"] = var or "0"  # read at the library's first decode
        assert fn(blob.data_ptr(), C.addressof(h), 0, 1, out.data_ptr(), st.cuda_stream, None) == 0
        torch.cuda.synchronize()
        assert torch.equal(out[: a.ffn * a.hidden], src[: a.ffn * a.hidden]), f"{spec}: decode mismatch"
        g0 = h.seg
        libs.append((fn, blob, h, int(g0[1].off_lut) + 2 * int(g0[0].n)))
    for r in range(reps):
        for i, (fn, blob, h, _) in enumerate(libs):
            assert fn(blob.data_ptr(), C.addressof(h), 0, 1, out.data_ptr(), st.cuda_stream,
                      spans[i, r].data_ptr()) == 0
            torch.cuda._sleep(100000)
    torch.cuda.synchronize()
    sp = spans.cpu().numpy()
    peak = 6556.2
    for i, p in enumerate(paths):
        alg = libs[i][3]
        us = float(np.median(sp[i, 3:, 1] - sp[i, 3:, 0])) / 1e3
        print(json.dumps({"lib": p, "device_us": round(us, 2), "gbs": round(alg / us / 1e3, 1),
                          "frac": round(alg / us / 1e3 / peak, 3)}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
