#!/bin/bash
# K9 / pre-MoE block A/B on one box (run under gpurun from the repo root):
# the in-tree build (with and without PDL) against _variants/base.so, then
# the kernel parity tests on the in-tree build.
mkdir -p gpurun_out
cp paper_2510_10302_b200/libspmoe.so /tmp/new.so
for v in new nopdl base new nopdl base; do
  if [ $v = base ]; then cp _variants/base.so paper_2510_10302_b200/libspmoe.so; else cp /tmp/new.so paper_2510_10302_b200/libspmoe.so; fi
  echo "== $v"
  if [ $v = nopdl ]; then export SPMOE_NO_PDL=1; else unset SPMOE_NO_PDL; fi
  python tools/premoe_bench.py 5 200; python tools/premoe_bench.py 1 200
done
unset SPMOE_NO_PDL
cp /tmp/new.so paper_2510_10302_b200/libspmoe.so
timeout 600 python -m pytest tests/test_attn_gpu.py tests/test_kernels_gpu.py tests/test_e2e_gpu.py -q -m gpu -x 2>&1 | tail -2
