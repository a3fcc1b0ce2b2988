#!/bin/bash
# build, the full -m gpu suite, the headline bench line (XC tier) and the
# reference arm; outputs in gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/gt.log 2>&1; tail -3 gpurun_out/gt.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_xc.json 2> gpurun_out/bench_xc.err; tail -2 gpurun_out/bench_xc.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_xc.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value", "tpot_ms", "acceptance_rate", "h2d_gbs", "ms_per_step", "cutoff_layer")})
for k in ("roofline_k3", "roofline_decode"):
    r = d.get(k) or {}
    print(k, r.get("frac"), r.get("ms_per_launch"), (r.get("cuda_events") or {}).get("frac"), r.get("by_shape"))
print("e2e", d["e2e"]["value"], "cpu", (d.get("cpu_baseline") or {}).get("value"))
PY
