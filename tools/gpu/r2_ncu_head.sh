mkdir -p gpurun_out/r2
timeout 600 ncu --profile-from-start off -k regex:k_head_bwd --set full --clock-control none --import-source on \
  -o gpurun_out/r2/head_bwd python tools/ncu_step.py --map gpurun_out/r2/head_map.json > gpurun_out/r2/ncu_head.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r2/head_bwd.ncu-rep --page details --csv > gpurun_out/r2/head_bwd.details.csv 2>&1
ncu -i gpurun_out/r2/head_bwd.ncu-rep --page raw --csv > gpurun_out/r2/head_bwd.raw.csv 2>&1
ncu -i gpurun_out/r2/head_bwd.ncu-rep --page source --csv > gpurun_out/r2/head_bwd.source.csv 2>&1
rm -f gpurun_out/r2/head_bwd.ncu-rep
grep -E "Duration|DRAM Throughput|Memory Throughput|Issue Slots Busy|Achieved Occupancy|Registers Per|Eligible|No Eligible|Theoretical Occ" gpurun_out/r2/head_bwd.details.csv | head -20
