#!/bin/bash
# ncu: DRAM traffic of single-expert K3 launches (tc T=2, cuda-core T=1) + the XC decode kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/k3_single_tc.csv python tools/k3_single.py 4 20000 2 tc > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/k3_single_cc.csv python tools/k3_single.py 4 20000 1 cuda_core > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:xc_decode -s 2 -c 1 -o gpurun_out/xc_decode_final python -m pytest tests/test_codec.py -q -m gpu -k full_mixtral > gpurun_out/ncu_dec.log 2>&1
ls -la gpurun_out/*.csv gpurun_out/xc_decode_final.ncu-rep
