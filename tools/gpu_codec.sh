#!/bin/bash
# Codec check (run under gpurun from the repo root): build, the XC tests,
# the decode timing tool for both register budgets (3 / 2 CTAs per SM).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_codec.py -q -m gpu -x > gpurun_out/gt_codec.log 2>&1; tail -3 gpurun_out/gt_codec.log
for c in ${VARIANTS:-0 3}; do
  echo "variant=$c"; SPMOE_XC_DEC=$c timeout 300 python tools/decode_insitu.py 2>&1 | tail -6
done
