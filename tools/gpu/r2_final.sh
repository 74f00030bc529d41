mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2/smoke.log
timeout 600 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2/bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value']/1e6, d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline']['attainable_frac'], d['halo']['share'], d['clocks'])
PY
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2/bench_ref.json 2> gpurun_out/r2/bench_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/r2/bench_ref.json
