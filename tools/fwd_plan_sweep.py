"""Sweep the general forward kernel's plan (MB tiles per unit, accumulator sets, split-K cap)
for one shape and compare with the planner's own choice.  Args: cin:cout:D:HW[:dgrad] ..."""
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
    f = spec.split(":")
    ci, co, d, e = (int(v) for v in f[:4])
    dgrad = len(f) > 4 and f[4] == "dgrad"
    x = Slab(1, ci, d, e, e, torch.bfloat16, "cuda")
    y = Slab(1, co, d, e, e, torch.bfloat16, "cuda")
    x.storage.normal_()
    w = torch.randn(27 * ci * co, device="cuda") * 0.05
    b = torch.zeros(co, device="cuda")
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())
    nb = _lib.call_size("vm_conv3d_fwd_tc_ws_bytes", 1, ci, co, d, e, e)
    ws = torch.zeros(max(nb, 16) // 4 + 64, device="cuda")
    flops = 2.0 * 27 * ci * co * d * e * e

    def fn():
        _lib.call("vm_conv3d_fwd_tc_ws", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride, None, 0,
                  1, ci, co, d, e, e, 1, _lib.ptr(ws), nb, _lib.stream_ptr())

    lib.vm_debug_set_fwd_plan(0, 0)
    lib.vm_debug_set_fwd_max_split(16)
    t0 = timed(fn)
    ref = y.storage.clone()
    res = []
    for mb in range(1, 9):
        for acc in (1, 3):
            for ms in (1, 2, 3, 4, 6, 9, 12):
                lib.vm_debug_set_fwd_plan(mb, acc)
                lib.vm_debug_force_fwd_split(ms)
                try:
                    t = timed(fn)
                except Exception as ex:  # noqa: BLE001
                    continue
                ok = torch.equal(y.storage, ref) or float((y.storage.float() - ref.float()).abs().max()) < 0.1
                res.append((t, mb, acc, ms, ok))
    lib.vm_debug_set_fwd_plan(0, 0)
    lib.vm_debug_force_fwd_split(0)
    res.sort()
    print(f"{ci}->{co} @{d}x{e}^2: planner {t0:.1f} us ({flops / t0 / 1e6:.0f} TF/s); best:", flush=True)
    for t, mb, acc, ms, ok in res[:6]:
        print(f"   MB={mb} nacc={acc} split={ms}: {t:.1f} us ({flops / t / 1e6:.0f} TF/s) ok={ok}", flush=True)
