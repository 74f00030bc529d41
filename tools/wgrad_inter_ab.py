"""A/B: wgrad K stages interleaved over the split CTAs vs contiguous ranges, alternating the two
settings per shape (best of 3 each: the box drifts over a run).  Forces the planner flag
(vm_debug_set_wgrad_interleave: 0 never, 1 size-gated default, 2 always)."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
specs = sys.argv[1:] or ["16:16:128", "48:16:128", "32:32:64", "64:64:32", "32:32:256", "96:32:256", "64:64:128",
                         "192:64:128"]
for spec in specs:
    ci, co, e = (int(v) for v in spec.split(":"))
    x = Slab(1, ci, e, e, e, torch.bfloat16, "cuda")
    g = Slab(1, co, e, e, e, torch.bfloat16, "cuda")
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device="cuda")
    gb = torch.zeros(co, device="cuda")
    ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device="cuda")

    def run():
        _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb),
                  _lib.ptr(ws), 1, ci, co, e, e, e, _lib.stream_ptr())

    best = {0: 1e9, 2: 1e9}
    for rep in range(3):
        for v in (0, 2):
            lib.vm_debug_set_wgrad_interleave(v)
            for _ in range(2):
                run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                run()
            b.record()
            torch.cuda.synchronize()
            best[v] = min(best[v], a.elapsed_time(b) / 5 * 1e3)
    print(f"{ci:4d}->{co:4d} @{e}^3: contiguous {best[0]:8.1f} us  interleaved {best[2]:8.1f} us  "
          f"({best[0] / best[2]:.3f}x)", flush=True)
lib.vm_debug_set_wgrad_interleave(1)
