#!/bin/bash
# bench with decode roofline + XC-tier sweeps of configs #3 / #4 (+ Mixtral policies)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_codec.py -q -m gpu -x 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xc2.json 2> gpurun_out/bench_xc2.err
python -c "import json; d=json.loads(open('gpurun_out/bench_xc2.json').read().strip().splitlines()[-1]); print(d['value'], d['tpot_ms'], d['acceptance_rate'], d['roofline']['frac'], d['roofline_decode'])"
rm -f gpurun_out/sweeps_xc.jsonl
timeout 1500 python tools/sweeps.py deepseek --out gpurun_out/sweeps_xc.jsonl --steps 6 > /dev/null 2> gpurun_out/sw_ds.err; tail -1 gpurun_out/sw_ds.err
timeout 1200 python tools/sweeps.py qwen --out gpurun_out/sweeps_xc.jsonl --steps 6 > /dev/null 2> gpurun_out/sw_qw.err; tail -1 gpurun_out/sw_qw.err
timeout 1200 python tools/sweeps.py mixtral --out gpurun_out/sweeps_xc.jsonl --steps 6 > /dev/null 2> gpurun_out/sw_mx.err; tail -1 gpurun_out/sw_mx.err
wc -l gpurun_out/sweeps_xc.jsonl
