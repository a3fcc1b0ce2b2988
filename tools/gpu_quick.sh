#!/bin/bash
# Quick GPU check (run under gpurun from the repo root): build, codec tests,
# decode timing, one short bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_codec.py -q -m gpu -x 2>&1 | tail -2
python tools/decode_ab.py paper_2510_10302_b200/libspmoe.so
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value", "tpot_ms", "acceptance_rate", "h2d_gbs", "h2d_expert_gbs", "ms_per_step")})
for k in ("roofline", "roofline_k3"):
    r = d[k]
    print(k, round(r["frac"], 3), round(r["ms_per_launch"] * 1e3, 1), "us", (r.get("cuda_events") or {}).get("frac"))
print(d["host_codec"])
PY
