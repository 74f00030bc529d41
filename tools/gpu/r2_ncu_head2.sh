mkdir -p gpurun_out/r2
timeout 600 ncu -k regex:k_head_bwd_team -c 1 --set full --clock-control none --import-source on \
  -o gpurun_out/r2/head_team python tools/head_ab.py 16:128 > gpurun_out/r2/ncu_head2.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r2/head_team.ncu-rep --page details --csv > gpurun_out/r2/head_team.details.csv 2>&1
ncu -i gpurun_out/r2/head_team.ncu-rep --page raw --csv > gpurun_out/r2/head_team.raw.csv 2>&1
rm -f gpurun_out/r2/head_team.ncu-rep
grep -E "\"Duration|DRAM Throughput|Issue Slots Busy|Achieved Occupancy|Eligible Warps|No Eligible" gpurun_out/r2/head_team.details.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
