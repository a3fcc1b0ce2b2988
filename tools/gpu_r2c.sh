#!/bin/bash
# codec tests + bench (XC) with K3 breakdown
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_codec.py tests/test_engine_gpu.py -q -m gpu -x > gpurun_out/codec.log 2>&1; tail -3 gpurun_out/codec.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xc.json 2> gpurun_out/bench_xc.err; tail -2 gpurun_out/bench_xc.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_xc.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value", "tpot_ms", "acceptance_rate", "tokens_emitted", "h2d_gbs", "h2d_expert_gbs", "ms_per_step", "cutoff_layer")})
print(d["roofline"]["frac"], d["roofline"]["by_shape"])
PY
