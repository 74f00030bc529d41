mkdir -p gpurun_out/r3
timeout 900 python bench.py --no-cpu --emulate-config cfg4 --steps 5 --warmup 3 > gpurun_out/r3/emu_cfg4.json 2> gpurun_out/r3/emu_cfg4.err; echo "emu rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r3/emu_cfg4.json').read().strip().splitlines()[-1]); h=d['halo']
print({k:h.get(k) for k in ('share','ms_step','ms_nohalo','bytes_per_step_rank','projected_share_no_overlap','transport','rounds_ms')})
PY
tail -3 gpurun_out/r3/emu_cfg4.err
timeout 900 python bench.py --config cfg3 --scaling-base on --no-cpu --no-emulate --steps 5 --warmup 3 > gpurun_out/r3/cfg3_base.json 2> gpurun_out/r3/cfg3_base.err; echo "cfg3 rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r3/cfg3_base.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value']/1e6, d.get('scaling_base'), d['parity'])
PY
tail -3 gpurun_out/r3/cfg3_base.err
