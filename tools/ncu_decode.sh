#!/bin/bash
# ncu --set full of one XC segment decode launch (tools/decode_insitu.py's
# back-to-back mode); report in gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xc_decode -s 5 -c 1 \
  -o gpurun_out/ncu_decode -f python tools/decode_insitu.py > gpurun_out/ncu_decode.log 2>&1
tail -3 gpurun_out/ncu_decode.log
