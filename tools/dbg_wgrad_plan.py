"""In-graph time of the general weight-gradient kernel per forced plan (runs, KS, M-tiles per
CTA; vm_debug_force_wgrad_plan) against the planner's choice."""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
SH = [(64, 64, 32), (32, 64, 32), (192, 64, 32), (128, 128, 16), (64, 128, 16), (64, 64, 64), (128, 64, 32)]
for (ci, co, e) in SH:
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
    g = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device='cuda')
    gb = torch.zeros(co, device='cuda')
    res = {}
    for key in [(2, 0, 0)] + [(r, ks, m) for r in (0, 1) for ks in (0, 64, 128, 256) for m in (1, 2)]:
        lib.vm_debug_force_wgrad_plan(*key)  # (2, 0, 0): general kernel, planner's choice
        try:
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
            res[key] = e0.elapsed_time(e1) * 1e3 / 50
        except Exception:
            pass
    lib.vm_debug_force_wgrad_plan(-1, 0, 0)
    auto = res.get((2, 0, 0), float('nan'))
    best = min((v, k) for k, v in res.items() if k != (2, 0, 0))
    print(f"{ci}->{co} @{e}^3: auto {auto:.1f} us, best {best[0]:.1f} us at (runs, KS, mpu) = {best[1]}")
