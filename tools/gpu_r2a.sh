#!/bin/bash
# XC host tier: codec tests, full GPU suite, bench with XC and raw tiers
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_codec.py -q -m gpu -s > gpurun_out/codec.log 2>&1; tail -5 gpurun_out/codec.log
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/gt.log 2>&1; tail -5 gpurun_out/gt.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_xc.json 2> gpurun_out/bench_xc.err; tail -3 gpurun_out/bench_xc.err
timeout 900 python bench.py --steps 10 --warmup 3 --host-codec none --no-cpu-baseline > gpurun_out/bench_raw.json 2> gpurun_out/bench_raw.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_xc.json", "gpurun_out/bench_raw.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, {k: d.get(k) for k in ("value", "tpot_ms", "acceptance_rate", "tokens_emitted", "h2d_gbs", "h2d_expert_gbs", "host_codec", "hidden_prefetch_fraction", "cutoff_layer")}, d["roofline"]["frac"], d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e)
PY
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
echo done
