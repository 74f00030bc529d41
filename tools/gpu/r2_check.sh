set -x
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2/smoke.log
timeout 600 python bench.py > gpurun_out/r2/bench_default.json 2> gpurun_out/r2/bench_default.err; echo "bench rc=$?"
cat gpurun_out/r2/bench_default.json; tail -20 gpurun_out/r2/bench_default.err
