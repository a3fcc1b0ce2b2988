#!/bin/bash
# Codec check (run under gpurun from the repo root): build, the XC tests and
# the decode timing tool (device clock: back to back, rotating buffers, idle
# gaps, a concurrent H2D copy).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_codec.py -q -m gpu -x > gpurun_out/gt_codec.log 2>&1; tail -3 gpurun_out/gt_codec.log
timeout 300 python tools/decode_insitu.py 2>&1 | tail -6
