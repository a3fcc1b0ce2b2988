#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/gt.log 2>&1; tail -4 gpurun_out/gt.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
