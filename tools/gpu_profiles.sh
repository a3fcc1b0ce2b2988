#!/bin/bash
# Round-2 profile captures (run under gpurun from the repo root; one GPU):
#   decode DRAM traffic per launch (bench launch shape) -> profiles JSON
#   K3 unit-kernel DRAM traffic per single-expert call    -> profiles JSON
#   ncu --set full of one W1|W3 decode launch and of one single-expert K3 unit launch
#   k3_single timings (device clock) alone / under an H2D copy
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M -k regex:xc_decode --csv --log-file gpurun_out/decode_traffic.csv \
  python tools/decode_traffic.py run > gpurun_out/decode_traffic_run.json 2>gpurun_out/decode_traffic.err
ALG=$(python -c "import json;print(json.dumps(json.loads(open('gpurun_out/decode_traffic_run.json').read().strip().splitlines()[-1])['algorithmic_bytes_per_segment']))")
python tools/decode_traffic.py parse gpurun_out/decode_traffic.csv gpurun_out/ncu_xc_decode_traffic.json "$ALG" | head -8
timeout 600 ncu --metrics $M -k regex:"ffn_tc_unit|gather_rows|reduce_units" --csv --log-file gpurun_out/k3_traffic.csv \
  python tools/k3_single.py 4 20000 1,2 tc_units > gpurun_out/k3_traffic_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xc_decode -s 2 -c 1 \
  -o gpurun_out/ncu_decode_w13 -f python tools/decode_traffic.py run > gpurun_out/ncu_decode_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_tc_unit -s 3 -c 1 \
  -o gpurun_out/ncu_k3_unit_1x1 -f python tools/k3_single.py 4 20000 1 tc_units > gpurun_out/ncu_k3_full.log 2>&1
timeout 600 python tools/k3_single.py 20 20000 1,2,5 tc_units,tc,cuda_core > gpurun_out/k3_single.log 2>&1
timeout 600 python tools/k3_single.py 20 20000 1,2 tc_units,tc h2d >> gpurun_out/k3_single.log 2>&1
cat gpurun_out/k3_single.log
ls gpurun_out
