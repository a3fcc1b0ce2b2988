#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 8 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ffn_tc|ffn_kernel" -s 8 -c 6 -o gpurun_out/prof_tc python tools/bench_kernels.py --cases mixtral_T5 --iters 2 --warmup 2 > gpurun_out/ncu_tc.log 2>&1; tail -2 gpurun_out/ncu_tc.log
SPMOE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.json 2> gpurun_out/bench_ncu.err; tail -2 gpurun_out/bench_ncu.err
