"""A/B of wide weight gradients (Cout > 160): 128-channel output chunks as CTA columns of one
launch vs one call per chunk (alternating, best of 3).  Args: cin:cout:D:H:W ..."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
for spec in sys.argv[1:] or ["512:512:2:16:16", "256:256:4:32:32", "768:256:4:32:32", "512:512:16:16:16"]:
    ci, co, d, h, w = (int(v) for v in spec.split(":"))
    x = Slab(1, ci, d, h, w, torch.bfloat16, "cuda")
    g = Slab(1, co, d, h, w, torch.bfloat16, "cuda")
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device="cuda")
    gb = torch.zeros(co, device="cuda")
    nws = 0
    for v in (0, 1):
        lib.vm_debug_set_wgrad_merge(v)
        nws = max(nws, _lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, d, h, w))
    ws = torch.empty(nws // 4 + 64, device="cuda")
    best, outs = {}, {}
    for rep in range(3):
        for v in (0, 1):
            lib.vm_debug_set_wgrad_merge(v)
            run = lambda: _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw),  # noqa: E731
                                    _lib.ptr(gb), _lib.ptr(ws), 1, ci, co, d, h, w, _lib.stream_ptr())
            run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                run()
            b.record()
            torch.cuda.synchronize()
            best[v] = min(best.get(v, 1e9), a.elapsed_time(b) / 5 * 1e3)
            outs[v] = (gw.clone(), gb.clone())
    rel = float((outs[0][0] - outs[1][0]).norm() / outs[0][0].norm())
    relb = float((outs[0][1] - outs[1][1]).norm() / outs[0][1].norm())
    tf = 2 * 27 * ci * co * d * h * w / (best[1] * 1e-6) / 1e12
    print(f"{ci:4d}->{co:4d} @{d}x{h}x{w}: per-chunk calls {best[0]:7.1f} us  one launch {best[1]:7.1f} us "
          f"({best[0] / best[1]:.2f}x, {tf:.0f} TF/s)  rel diff gw {rel:.1e} gb {relb:.1e}", flush=True)
lib.vm_debug_set_wgrad_merge(1)
