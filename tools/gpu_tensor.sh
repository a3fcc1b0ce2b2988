#!/bin/bash
# Tensor-pipe evidence for K3 in the compute-heavier regime (run under gpurun):
# bench_kernels timings at T = 5 / 72 / 512 / 2048 routed tokens (Mixtral
# shapes, 8 experts), then ncu metrics of the tcgen05 kernels at each size.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
C=mixtral_T5,mixtral_T72,mixtral_T512,mixtral_T2048
timeout 900 python tools/bench_kernels.py --cases $C --iters 10 --warmup 3 --json gpurun_out/bench_kernels_tc.json > gpurun_out/bench_kernels_tc.log 2>&1
tail -4 gpurun_out/bench_kernels_tc.log | cut -c1-400
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active
timeout 1200 ncu --metrics $M -k regex:"ffn_tc_kernel" --csv --log-file gpurun_out/ncu_tc_tensor.csv \
  python tools/bench_kernels.py --cases $C --iters 1 --warmup 1 > gpurun_out/ncu_tc_tensor.log 2>&1
tail -2 gpurun_out/ncu_tc_tensor.log
