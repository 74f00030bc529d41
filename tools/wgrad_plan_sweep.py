"""Sweep the general weight-gradient plan (K chunk KS, minimum stages per K split) for one
shape, with and without the finalize (vm_debug_skip_wgrad_finalize: wrong results, timing
only).  Args: cin:cout:D:HW ..."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()


def timed(fn, reps=10):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / reps * 1e3)
    return best


for spec in sys.argv[1:]:
    ci, co, d, e = (int(v) for v in spec.split(":"))
    x = Slab(1, ci, d, e, e, torch.bfloat16, "cuda")
    g = Slab(1, co, d, e, e, torch.bfloat16, "cuda")
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device="cuda")
    gb = torch.zeros(co, device="cuda")
    flops = 2.0 * 27 * ci * co * d * e * e
    out = []
    for ks in (0, 64, 128, 192, 256):
        for spk in (1, 2, 3, 4, 6, 8, 1000):
            lib.vm_debug_force_wgrad_plan(-1, ks, 0)
            lib.vm_debug_set_wgrad_min_spk(spk)
            try:
                ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, d, e, e) // 4 + 64, device="cuda")
                fn = lambda: _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw),  # noqa: E731
                                       _lib.ptr(gb), _lib.ptr(ws), 1, ci, co, d, e, e, _lib.stream_ptr())
                t = timed(fn)
                lib.vm_debug_skip_wgrad_finalize(1)
                t_nf = timed(fn)
                lib.vm_debug_skip_wgrad_finalize(0)
            except Exception:  # noqa: BLE001
                lib.vm_debug_skip_wgrad_finalize(0)
                continue
            out.append((t, ks, spk, t_nf))
    lib.vm_debug_force_wgrad_plan(-1, 0, 0)
    lib.vm_debug_set_wgrad_min_spk(2)
    ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, d, e, e) // 4 + 64, device="cuda")
    t0 = timed(lambda: _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb),
                                 _lib.ptr(ws), 1, ci, co, d, e, e, _lib.stream_ptr()))
    out.sort()
    print(f"{ci}->{co} @{d}x{e}^2: planner {t0:.1f} us ({flops / t0 / 1e6:.0f} TF/s)", flush=True)
    for t, ks, spk, t_nf in out[:5]:
        print(f"   KS={ks} min_spk={spk}: {t:.1f} us ({flops / t / 1e6:.0f} TF/s), without finalize {t_nf:.1f} us", flush=True)
