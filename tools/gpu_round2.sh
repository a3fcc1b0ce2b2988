#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu > gpurun_out/kt.log 2>&1; tail -3 gpurun_out/kt.log
timeout 300 python tools/bench_kernels.py --cases mixtral_T5,mixtral_T1,mixtral_T9,deepseek_T5,qwen_T5 > gpurun_out/kb.log 2>&1; cat gpurun_out/kb.log | cut -c1-400
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -m gpu > gpurun_out/et.log 2>&1; tail -30 gpurun_out/et.log
timeout 900 python tools/tune_acceptance.py mixtral_8x7b '[{"expert_spread":0.05},{"expert_spread":0.05,"embed_std":1.0},{"expert_spread":0.2,"embed_std":1.0},{"expert_spread":0.5,"embed_std":1.0},{"expert_spread":0.2,"embed_std":0.3}]' 8 2>&1 | grep -E "arch|Error|error" | tail -12
