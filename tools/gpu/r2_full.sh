mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2/bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline_by_kind']['conv_wgrad'], d['roofline_by_kind']['conv_fwd'], d['roofline_by_kind']['conv_dgrad'])
h=d['halo']; print({k: h[k] for k in h if k != 'method'})
print(d['cpu_baseline'])
PY
