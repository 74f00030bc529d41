# end-of-round-2 evidence refresh (one GPU; each ncu command after its plain run exited 0)
set -x
O=gpurun_out/r2f
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,launch__registers_per_thread,sm__cycles_elapsed.avg.per_second
python bench.py --steps 2 --warmup 3 --no-cpu --no-emulate --no-graph > $O/plain_launch.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-emulate --no-graph > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/ncu_step.py --map $O/step_map_cfg2.json > /dev/null 2>&1 && \
timeout 900 ncu --profile-from-start off -k regex:^k_ --metrics $M --clock-control none \
  -o $O/step_cfg2 -f python tools/ncu_step.py --map $O/step_map_cfg2.json > $O/ncu_step2.log 2>&1; echo "step2 rc=$?"
python tools/ncu_summary.py $O/step_cfg2.ncu-rep $O/ncu_step_dram_cfg2.json --map $O/step_map_cfg2.json > /dev/null
rm -f $O/step_cfg2.ncu-rep
python tools/ncu_step.py --extent 256 --scale 0.5 --map $O/step_map_cfg3.json > /dev/null 2>&1 && \
timeout 1200 ncu --profile-from-start off -k regex:^k_ --metrics $M --clock-control none \
  -o $O/step_cfg3 -f python tools/ncu_step.py --extent 256 --scale 0.5 --map $O/step_map_cfg3.json > $O/ncu_step3.log 2>&1; echo "step3 rc=$?"
python tools/ncu_summary.py $O/step_cfg3.ncu-rep $O/ncu_step_dram_cfg3.json --map $O/step_map_cfg3.json > /dev/null
rm -f $O/step_cfg3.ncu-rep
for spec in "fwd 64 64 32:k_conv_fwd_tc" "fwd 128 128 16:k_conv_fwd_tc"; do
  args=${spec%%:*}; k=${spec##*:}; set -- $args
  python tools/conv_one.py $1 $2 $3 $4 2 > /dev/null 2>&1 && \
  timeout 400 ncu --set full --import-source on --clock-control none -k "regex:${k}" -s 1 -c 1 \
    -o $O/full_${1}_${2}_${3}_${4} -f python tools/conv_one.py $1 $2 $3 $4 2 > $O/ncu_full_${1}_${2}_${4}.log 2>&1
  echo "full $spec rc=$?"
  R=$O/full_${1}_${2}_${3}_${4}
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
  rm -f $R.ncu-rep
done
python tools/halo26_probe.py 32:256 > /dev/null 2>&1 && \
timeout 300 ncu --set full --clock-control none -k regex:k_slab_boxes -s 4 -c 2 -o $O/full_boxes -f \
  python tools/halo26_probe.py 32:256 > $O/ncu_boxes.log 2>&1; echo "boxes rc=$?"
ncu -i $O/full_boxes.ncu-rep --page raw --csv > $O/full_boxes.raw.csv 2>/dev/null; rm -f $O/full_boxes.ncu-rep
du -sh gpurun_out; ls -la $O/
