"""In-graph time of vm_conv3d_wgrad_tc on the kd-along-N shapes: straight-line (templated)
MMA issue vs the runtime-bounded loop (vm_debug_set_wgrad_kd_runtime)."""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
SHAPES = [(16, 16, 128), (48, 16, 128), (1, 16, 128), (32, 32, 64), (96, 32, 64), (16, 32, 64)]
for (ci, co, e) in SHAPES:
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
    g = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device='cuda')
    gb = torch.zeros(co, device='cuda')
    ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device='cuda')
    res, outs = {}, {}
    mode = sys.argv[1] if len(sys.argv) > 1 else "runtime"
    for rt in ((1, 0) if mode == "runtime" else (4, 3, 2)):
        if mode == "runtime":
            lib.vm_debug_set_wgrad_kd_runtime(rt)
        else:
            lib.vm_debug_set_wgrad_ksub_stages(rt)
        # the workspace depends on the plan (cluster mode keeps one partial per 8 CTAs)
        ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device='cuda')

        def run():
            _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb),
                      _lib.ptr(ws), 1, ci, co, e, e, e, _lib.stream_ptr())
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            run()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(10):
                    run()
        gr.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        res[rt] = e0.elapsed_time(e1) * 1e3 / 50
        outs[rt] = (gw.clone(), gb.clone())
    lib.vm_debug_set_wgrad_kd_runtime(0)
    lib.vm_debug_set_wgrad_ksub_stages(2)
    if mode == "runtime":
        same = torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
        print(f"{ci}->{co} @{e}^3: runtime loop {res[1]:.1f} us, straight-line {res[0]:.1f} us, bitwise same {same}")
    else:
        print(f"{ci}->{co} @{e}^3: ksub min-stages 4/3/2: {res[4]:.1f} / {res[3]:.1f} / {res[2]:.1f} us")
