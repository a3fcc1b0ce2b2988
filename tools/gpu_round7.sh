#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --write-calibration > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json; cp profiles/bench_calibration.json gpurun_out/
rm -f gpurun_out/sweeps.jsonl
timeout 900 python tools/sweeps.py mixtral --out gpurun_out/sweeps.jsonl 2>&1 | grep -v "^{" | tail -3
timeout 900 python tools/sweeps.py deepseek --out gpurun_out/sweeps.jsonl 2>&1 | grep -v "^{" | tail -3
timeout 900 python tools/sweeps.py qwen --out gpurun_out/sweeps.jsonl 2>&1 | grep -v "^{" | tail -3
python -c "
import json
for l in open('gpurun_out/sweeps.jsonl'):
    r=json.loads(l); print(r['sweep'], r['point'], 'cut',r['cutoff'], 'tpot %.1f'%r['tpot_ms'], 'tok/s %.2f'%r['tokens_per_s'], 'hit %.3f'%r['hit_rate'], 'acc %.2f'%r['acceptance'], 'hid', r['hidden_prefetch_fraction'])
"
