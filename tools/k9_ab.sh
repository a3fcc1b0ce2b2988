#!/bin/bash
mkdir -p gpurun_out
cp paper_2510_10302_b200/libspmoe.so /tmp/new.so
for v in new base new base; do
  if [ $v = new ]; then cp /tmp/new.so paper_2510_10302_b200/libspmoe.so; else cp _variants/base.so paper_2510_10302_b200/libspmoe.so; fi
  echo "== $v"; python tools/premoe_bench.py 5 200; python tools/premoe_bench.py 1 200
done
cp /tmp/new.so paper_2510_10302_b200/libspmoe.so
timeout 600 python -m pytest tests/test_attn_gpu.py tests/test_kernels_gpu.py -q -m gpu -x 2>&1 | tail -2
