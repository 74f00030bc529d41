set -x
mkdir -p gpurun_out/r2
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu --layer-csv gpurun_out/r2/cfg3_layers.csv > gpurun_out/r2/bench_cfg3.json 2> gpurun_out/r2/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-emulate --layer-csv gpurun_out/r2/cfg2_layers.csv > gpurun_out/r2/bench_cfg2_layers.json 2> gpurun_out/r2/bench_cfg2_layers.err; echo "cfg2 rc=$?"
for spec in "wgrad 32 32 256" "wgrad 16 16 128" "fwd 32 32 256" "fwd 16 16 128"; do
  set -- $spec
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_conv_(wgrad_kd|fwd_sweep)" -s 2 -c 1 \
    -o gpurun_out/r2/full_$1_$2_$3_$4 -f python tools/conv_one.py $1 $2 $3 $4 3 > gpurun_out/r2/ncu_$1_$2_$4.log 2>&1; echo "ncu $spec rc=$?"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-emulate --no-graph > gpurun_out/r2/ncu_launch.log 2>&1; echo "launch rc=$?"
