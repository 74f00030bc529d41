set -x
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 --layer-csv gpurun_out/r2/cfg2_layers.csv > gpurun_out/r2/bench_cfg2.json 2> gpurun_out/r2/bench_cfg2.err
python bench.py --steps 5 --warmup 3 --extent 256 --scale 0.5 --layer-csv gpurun_out/r2/cfg3_layers.csv > gpurun_out/r2/bench_cfg3.json 2> gpurun_out/r2/bench_cfg3.err
python -m pytest tests -x -q -m gpu > gpurun_out/r2/pytest_gpu.log 2>&1; tail -3 gpurun_out/r2/pytest_gpu.log
nproc; lscpu | head -20 > gpurun_out/r2/lscpu.txt
