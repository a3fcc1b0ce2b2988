#!/bin/bash
# Gated-draft check (run under gpurun): build, the Qwen-shaped parity tests
# (tiny_qwen engine vs oracle; real-shape end-to-end vs the CPU SD loop),
# then the Qwen / DeepSeek / Mixtral acceptance on short bench runs.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_e2e_gpu.py -q -m gpu -x -k "qwen" 2>&1 | tail -3
for c in qwen; do
  timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --no-event-pass > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', {k: d.get(k) for k in ('value','tpot_ms','acceptance_rate','hit_rate','hidden_prefetch_fraction','cutoff_layer')})"
done
