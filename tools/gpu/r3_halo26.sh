mkdir -p gpurun_out/r3
timeout 600 python -m pytest tests/test_gpu_nccl.py -x -q -p no:cacheprovider 2>&1 | tail -4
for ph in 1 3; do
VOXMESH_HALO_PHASES=$ph timeout 900 python bench.py --no-cpu --emulate-config cfg4 --steps 5 --warmup 3 > gpurun_out/r3/emu_cfg4_p$ph.json 2> gpurun_out/r3/emu_cfg4_p$ph.err; echo "emu phases=$ph rc=$?"
python - <<PY
import json
d=json.loads(open('gpurun_out/r3/emu_cfg4_p$ph.json').read().strip().splitlines()[-1]); h=d['halo']
print({k:h.get(k) for k in ('share','ms_step','ms_nohalo','bytes_per_step_rank','rounds_ms')})
PY
done
