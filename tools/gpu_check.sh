#!/bin/bash
# Targeted GPU check (run under gpurun from the repo root): build, the new /
# changed GPU tests, the end-to-end parity tests with their tolerance report
# (-s), compute-sanitizer racecheck + synccheck on the tiny engine test, smoke.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_facade.py tests/test_engine_gpu.py tests/test_native_abi.py -q -m gpu -x > gpurun_out/gt_new.log 2>&1; tail -3 gpurun_out/gt_new.log
timeout 1200 python -m pytest tests/test_e2e_gpu.py -q -m gpu -s > gpurun_out/gt_e2e.log 2>&1; tail -3 gpurun_out/gt_e2e.log; grep -a "max|dlogit|" gpurun_out/gt_e2e.log
for tool in racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python -m pytest tests/test_engine_gpu.py -q -m gpu -x \
    -k "tiny_draft_prefetch or test_engine_tiny_baseline_policies" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -a "ERROR SUMMARY\|passed\|failed" gpurun_out/sanitizer_$tool.log | tail -3
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
echo done
