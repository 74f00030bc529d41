mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2/pytest_gpu.log
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2/bench_cfg3.json 2> gpurun_out/r2/bench_cfg3.err; echo "cfg3 rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2/bench_cfg3.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value']/1e6, d['roofline']['kernel'], d['roofline']['frac'], d['roofline'].get('attainable_frac'), d.get('halo', {}).get('share'), d['clocks'])
print({k: (v.get('frac'), v.get('attainable_frac')) for k, v in d['roofline_by_kind'].items() if k.startswith('conv')})
PY
