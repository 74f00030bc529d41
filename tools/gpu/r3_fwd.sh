# general fwd planner/drain change: parity + probes + per-shape timing
mkdir -p gpurun_out/r3
timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_guard.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/dbg_fwd_probe.py 2>&1 | grep "split=1 flags 0x1:"
python tools/conv_time.py fwd:64:64:32 fwd:128:128:16 fwd:64:128:16 fwd:192:64:32 fwd:32:64:32 dgrad:64:64:32 dgrad:128:128:16 fwd:384:128:32 fwd:128:64:32 2>&1 | tail -9
