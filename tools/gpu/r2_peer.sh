mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_peer_halo.py tests/test_gpu_nccl.py tests/test_gpu_conv.py -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2/bench_peer.json 2> gpurun_out/r2/bench_peer.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2/bench_peer.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ms_per_step'], json.dumps(d.get('halo'), indent=0))
PY
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --emulate-transport nccl 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nccl', d['halo']['share'], d['halo']['ms_step'], d['halo']['ms_nohalo'])"
