#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_tc_gpu.py -x -q -m gpu > gpurun_out/et.log 2>&1; tail -25 gpurun_out/et.log
timeout 900 python tools/tune_acceptance.py mixtral_8x7b '[{"expert_spread":0.02},{"expert_spread":0.05},{"expert_spread":0.1},{"expert_spread":0.05,"embed_std":1.0},{"expert_spread":0.05,"residual_scale":0.05}]' 8 2>&1 | grep -E "arch|Error|Traceback" | tail -12
