mkdir -p gpurun_out/r3
timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_guard.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/dbg_fwd_plan.py 2>&1 | tail -8 | cut -c1-90
timeout 600 python bench.py --no-cpu --no-emulate > gpurun_out/r3/b2.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r3/b2.json').read().strip().splitlines()[-1]); print('cfg2', d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_ms_per_step'])"
timeout 600 python bench.py --config cfg3 --no-cpu --no-emulate --steps 10 > gpurun_out/r3/b3.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r3/b3.json').read().strip().splitlines()[-1]); print('cfg3', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks'])"
