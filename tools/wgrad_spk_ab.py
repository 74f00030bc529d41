"""A/B of the general weight-gradient K split (vm_debug_set_wgrad_min_spk: minimum K stages per
split; large = no split) on deep-level shapes: python tools/wgrad_spk_ab.py Cin:Cout:D:HW ..."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
for spec in sys.argv[1:]:
    ci, co, d, e = (int(v) for v in spec.split(":"))
    x = Slab(1, ci, d, e, e, torch.bfloat16, "cuda")
    g = Slab(1, co, d, e, e, torch.bfloat16, "cuda")
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device="cuda")
    gb = torch.zeros(co, device="cuda")
    res = {}
    for spk in (2, 4, 8, 1000):
        lib.vm_debug_set_wgrad_min_spk(spk)
        ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, d, e, e) // 4 + 64, device="cuda")
        run = lambda: _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw),  # noqa: E731
                                _lib.ptr(gb), _lib.ptr(ws), 1, ci, co, d, e, e, _lib.stream_ptr())
        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            run()
        b.record()
        torch.cuda.synchronize()
        res[spk] = a.elapsed_time(b) / 5 * 1e3
    lib.vm_debug_set_wgrad_min_spk(2)
    print(f"{ci:4d}->{co:4d} @{d}x{e}^2: " + "  ".join(f"min_spk {k}: {v:7.1f} us" for k, v in res.items()), flush=True)
