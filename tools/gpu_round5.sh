#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/gt.log 2>&1; tail -4 gpurun_out/gt.log
timeout 300 python tools/bench_kernels.py --cases mixtral_T5,mixtral_T1,mixtral_T72,deepseek_T5,qwen_T5,qwen_T72 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except: print(l[:200]); continue
    print(r['name'], {k:(round(v['GBps']),round(v['ms']*1000)) for k,v in r.items() if isinstance(v,dict)})"
timeout 900 python bench.py --steps 8 --warmup 3 --write-calibration > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json; cp profiles/bench_calibration.json gpurun_out/ 2>/dev/null
timeout 1200 python tools/sweeps.py deepseek --out gpurun_out/sweeps.jsonl 2>&1 | tail -12
