"""A/B of the input-channel chunks of multi-group kd weight gradients (alternating, best of 3)."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
for spec in sys.argv[1:] or ["96:32:256", "96:32:64", "64:32:128", "48:16:128"]:
    ci, co, e = (int(v) for v in spec.split(":"))
    x = Slab(1, ci, e, e, e, torch.bfloat16, "cuda")
    g = Slab(1, co, e, e, e, torch.bfloat16, "cuda")
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device="cuda")
    gb = torch.zeros(co, device="cuda")
    ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device="cuda")
    best, outs = {}, {}
    for rep in range(3):
        for v in (0, 1):
            lib.vm_debug_set_wgrad_chunk(v)
            run = lambda: _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw),  # noqa: E731
                                    _lib.ptr(gb), _lib.ptr(ws), 1, ci, co, e, e, e, _lib.stream_ptr())
            run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                run()
            b.record()
            torch.cuda.synchronize()
            best[v] = min(best.get(v, 1e9), a.elapsed_time(b) / 3 * 1e3)
            outs[v] = (gw.clone(), gb.clone())
    rel = float((outs[0][0] - outs[1][0]).norm() / outs[0][0].norm())
    relb = float((outs[0][1] - outs[1][1]).norm() / outs[0][1].norm())
    print(f"{ci:4d}->{co:4d} @{e}^3: one call {best[0]:8.1f} us  chunked {best[1]:8.1f} us ({best[0] / best[1]:.2f}x)"
          f"  rel diff gw {rel:.1e} gb {relb:.1e}", flush=True)
lib.vm_debug_set_wgrad_chunk(1)
