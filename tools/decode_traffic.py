"""DRAM traffic of the XC decode kernel in the bench's launch shape (one
launch per segment of a Mixtral-8x7B expert, as the runtime issues them)
against its algorithmic bytes (segment code + sign|mantissa bytes read once,
bf16 written once).

  python tools/decode_traffic.py run                 # the launches (run under ncu)
  python tools/decode_traffic.py parse CSV [OUT]     # ncu CSV -> profiles JSON

ncu command (one B200):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:xc_decode --csv --log-file gpurun_out/decode_traffic.csv \
      python tools/decode_traffic.py run
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

REPS = 4


def run():
    import torch

    from paper_2510_10302_b200 import _native
    from paper_2510_10302_b200 import codec as X
    from paper_2510_10302_b200.model import fill_expert_blob, get_arch

    a = get_arch("mixtral_8x7b")
    dev = torch.device("cuda", 0)
    src = torch.empty((a.expert_elems,), dtype=torch.bfloat16, device=dev)
    fill_expert_blob(src, a, 1234, 0)
    enc = X.XcEncoder(X.expert_segments(a.ffn, a.hidden), dev)
    hdr = enc.plan(src)
    blob = enc.encode(src, hdr).clone()
    out = torch.empty_like(src)
    lib = _native.load()
    s = torch.cuda.current_stream().cuda_stream
    alg = []
    for g in range(hdr.nseg):
        lo = 0 if g == 0 else hdr.seg[g].off_lut
        hi = hdr.seg[g + 1].off_lut if g + 1 < hdr.nseg else hdr.blob_bytes
        alg.append(int(hi - lo) + 2 * int(hdr.seg[g].n))
    for _ in range(REPS):
        for g in range(hdr.nseg):
            _native.check("spmoe_xc_decode_segments", lib.spmoe_xc_decode_segments(
                C.c_void_p(blob.data_ptr()), C.addressof(hdr), g, 1, C.c_void_p(out.data_ptr()), C.c_void_p(s)))
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), src.view(torch.int16)), "decode mismatch"
    print(json.dumps({"algorithmic_bytes_per_segment": alg, "reps": REPS}), flush=True)


def parse(csv_path, out_path=None):
    import csv

    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    hdr = rows[0]
    i_id, i_name, i_m, i_v = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    i_u = hdr.index("Metric Unit")
    per = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0}
    for r in rows[1:]:
        if "xc_decode" not in r[i_name]:
            continue
        v = float(r[i_v].replace(",", "")) * scale.get(r[i_u], 1.0)
        per.setdefault(r[i_id], {})[r[i_m]] = v
    launches = [per[k] for k in sorted(per, key=int)]
    dram = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in launches]
    us = [d["gpu__time_duration.sum"] for d in launches]
    return launches, dram, us, out_path


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        launches, dram, us, _ = parse(sys.argv[2])
        # the three segments' algorithmic bytes of the fixed expert (seed 1234, row 0)
        alg = json.loads(sys.argv[4]) if len(sys.argv) > 4 else None
        res = {"launches": len(launches), "traffic_per_launch_bytes": sum(dram) / len(dram),
               "us_cold_mean": sum(us) / len(us), "dram_bytes": dram, "us_cold": us,
               "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                         "-k regex:xc_decode python tools/decode_traffic.py run (per-segment launches of one "
                         "Mixtral-8x7B expert, as the runtime issues them)"}
        if alg:
            n = len(alg)
            mean_alg = sum(alg[i % n] for i in range(len(dram))) / len(dram)
            res["algorithmic_bytes_per_launch"] = mean_alg
            res["ratio"] = res["traffic_per_launch_bytes"] / mean_alg
        out = sys.argv[3] if len(sys.argv) > 3 else None
        txt = json.dumps(res, indent=1)
        if out:
            Path(out).write_text(txt)
        print(txt)
