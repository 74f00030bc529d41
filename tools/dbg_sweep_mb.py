"""In-graph time of the kd-stacked sweep conv per forced MB (vm_debug_set_sweep_mb)."""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
for (ci, co, e, dg) in [(16, 16, 128, 0), (16, 16, 128, 1), (32, 32, 64, 0), (32, 32, 64, 1), (48, 16, 128, 0),
                        (16, 48, 128, 1), (16, 32, 64, 0)]:
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
    y = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    y.storage.normal_()
    w = torch.randn(27 * ci * co, device='cuda') * 0.05
    b = torch.zeros(co, device='cuda')
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device='cuda')
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())
    res = {}
    knob = sys.argv[1] if len(sys.argv) > 1 else "mb"
    vals = (0, 1, 2, 3, 4) if knob == "mb" else (0, 4, 8, 12, 16, 24, 32)
    for mb in vals:
        if knob == "mb":
            lib.vm_debug_set_sweep_mb(mb)
        else:
            lib.vm_debug_set_sweep_s(mb)
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                def run():
                    if dg:
                        _lib.call("vm_conv3d_fwd_tc", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride,
                                  y.p(), y.bstride, 1, ci, co, e, e, e, 2 | 4, _lib.stream_ptr())
                    else:
                        _lib.call("vm_conv3d_fwd_tc", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride,
                                  None, 0, 1, ci, co, e, e, e, 1, _lib.stream_ptr())
                run()
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(10):
                        run()
            g.replay()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[mb] = f"{e0.elapsed_time(e1) * 1e3 / 50:.1f}"
        except Exception:
            res[mb] = "-"
    lib.vm_debug_set_sweep_mb(0)
    lib.vm_debug_set_sweep_s(0)
    print(f"{ci}->{co} @{e}^3 {'dgrad' if dg else 'fwd'} {knob} auto/" + "/".join(str(v) for v in vals[1:]) + " = "
          + " / ".join(res[m] for m in vals))
