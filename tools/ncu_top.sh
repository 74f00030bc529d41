#!/bin/bash
# Full ncu capture (--set full, source) of one launch of the dominant kernel class in the
# cfg2 step (the level-0 16->16 weight-gradient kernel), summarised for profiles/.
set -e
python tools/conv_one.py wgrad 16 16 128 3
timeout 500 ncu --set full --import-source on --clock-control none -k regex:k_conv_wgrad_kd -s 2 -c 1 \
  -o gpurun_out/wgrad_kd_full -f python tools/conv_one.py wgrad 16 16 128 3 > gpurun_out/ncu_wgrad.log 2>&1
python tools/ncu_summary.py gpurun_out/wgrad_kd_full.ncu-rep gpurun_out/ncu_full_wgrad_kd.json > /dev/null
ncu -i gpurun_out/wgrad_kd_full.ncu-rep --page details --csv > gpurun_out/ncu_full_wgrad_kd_details.csv 2>/dev/null
python tools/conv_one.py fwd 16 16 128 3
timeout 500 ncu --set full --import-source on --clock-control none -k regex:k_conv_fwd_sweep -s 2 -c 1 \
  -o gpurun_out/sweep_full -f python tools/conv_one.py fwd 16 16 128 3 > gpurun_out/ncu_sweep.log 2>&1
python tools/ncu_summary.py gpurun_out/sweep_full.ncu-rep gpurun_out/ncu_full_sweep.json > /dev/null
ncu -i gpurun_out/sweep_full.ncu-rep --page details --csv > gpurun_out/ncu_full_sweep_details.csv 2>/dev/null
ls -la gpurun_out/*.ncu-rep
