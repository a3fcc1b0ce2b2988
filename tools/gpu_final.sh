bash tools/gpu_round.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_tc_unit -s 3 -c 1 -o gpurun_out/ncu_k3_unit_1x1 -f python tools/k3_single.py 4 20000 1 tc_units > gpurun_out/ncu_k3_full.log 2>&1
ncu -i gpurun_out/ncu_k3_unit_1x1.ncu-rep --page details --csv > gpurun_out/ncu_k3_details.csv 2>&1
ncu -i gpurun_out/ncu_k3_unit_1x1.ncu-rep --page raw --csv > gpurun_out/ncu_k3_raw.csv 2>&1
ls gpurun_out
