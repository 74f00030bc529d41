# round-2 evidence for profiles/r02 (one GPU; each ncu command after its plain run exited 0)
set -x
mkdir -p gpurun_out/r2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,launch__registers_per_thread,sm__cycles_elapsed.avg.per_second
# 1. launch list of the cfg2 bench (eager launches so every kernel is listed)
python bench.py --steps 2 --warmup 3 --no-cpu --no-emulate --no-graph > gpurun_out/r2/plain_launch.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-emulate --no-graph > gpurun_out/r2/ncu_launch.log 2>&1; echo "launch rc=$?"
# 2. per-launch DRAM traffic of one cfg2 step and one cfg3 step, attributed to step ops
python tools/ncu_step.py --map gpurun_out/r2/step_map_cfg2.json > /dev/null 2>&1 && \
timeout 900 ncu --profile-from-start off -k regex:^k_ --metrics $M --clock-control none \
  -o gpurun_out/r2/step_cfg2 -f python tools/ncu_step.py --map gpurun_out/r2/step_map_cfg2.json > gpurun_out/r2/ncu_step2.log 2>&1; echo "step2 rc=$?"
python tools/ncu_summary.py gpurun_out/r2/step_cfg2.ncu-rep gpurun_out/r2/ncu_step_dram_cfg2.json --map gpurun_out/r2/step_map_cfg2.json > /dev/null
rm -f gpurun_out/r2/step_cfg2.ncu-rep
python tools/ncu_step.py --extent 256 --scale 0.5 --map gpurun_out/r2/step_map_cfg3.json > /dev/null 2>&1 && \
timeout 1200 ncu --profile-from-start off -k regex:^k_ --metrics $M --clock-control none \
  -o gpurun_out/r2/step_cfg3 -f python tools/ncu_step.py --extent 256 --scale 0.5 --map gpurun_out/r2/step_map_cfg3.json > gpurun_out/r2/ncu_step3.log 2>&1; echo "step3 rc=$?"
python tools/ncu_summary.py gpurun_out/r2/step_cfg3.ncu-rep gpurun_out/r2/ncu_step_dram_cfg3.json --map gpurun_out/r2/step_map_cfg3.json > /dev/null
rm -f gpurun_out/r2/step_cfg3.ncu-rep
# 3. --set full of the dominant kernels
for spec in "wgrad 16 16 128:kd" "fwd 16 16 128:sweep" "fwd 48 16 128:sweepkw" "wgrad 32 32 256:kd" "fwd 32 32 256:sweep"; do
  args=${spec%%:*}; k=${spec##*:}; set -- $args
  python tools/conv_one.py $1 $2 $3 $4 2 > /dev/null 2>&1 && \
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k_conv_(wgrad_)?$k" -s 1 -c 1 \
    -o gpurun_out/r2/full_${1}_${2}_${3}_${4} -f python tools/conv_one.py $1 $2 $3 $4 2 > gpurun_out/r2/ncu_full_${1}_${2}_${4}.log 2>&1
  echo "full $spec rc=$?"
  R=gpurun_out/r2/full_${1}_${2}_${3}_${4}
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass > $R.source.csv 2>/dev/null
  rm -f $R.ncu-rep
done
python tools/push_time.py 32:32:256:256 > /dev/null 2>&1 && \
timeout 300 ncu --set full --clock-control none -k regex:k_depth_push -s 2 -c 1 -o gpurun_out/r2/full_push -f \
  python tools/push_time.py 32:32:256:256 > gpurun_out/r2/ncu_push.log 2>&1; echo "push rc=$?"
ncu -i gpurun_out/r2/full_push.ncu-rep --page raw --csv > gpurun_out/r2/full_push.raw.csv 2>/dev/null; rm -f gpurun_out/r2/full_push.ncu-rep
du -sh gpurun_out; ls -la gpurun_out/r2/
