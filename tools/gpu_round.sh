#!/bin/bash
# One GPU round: engine tests, bench, launch list, ncu of the K3 kernels.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -m gpu > gpurun_out/engine_tests.log 2>&1; tail -3 gpurun_out/engine_tests.log
timeout 900 python bench.py --steps 6 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
SPMOE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.json 2> gpurun_out/bench_ncu.err; tail -2 gpurun_out/bench_ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_ -s 6 -c 4 -o gpurun_out/prof_ffn python tools/bench_kernels.py --cases mixtral_T5 --iters 2 --warmup 3 > gpurun_out/ncu_ffn.log 2>&1; tail -3 gpurun_out/ncu_ffn.log
