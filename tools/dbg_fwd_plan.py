"""In-graph time of the general forward kernel per forced (MB, nacc) (vm_debug_set_fwd_plan)."""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
for (ci, co, e) in [(64, 64, 32), (32, 64, 32), (192, 64, 32), (128, 128, 16), (64, 128, 16), (96, 32, 64),
                    (32, 96, 64), (128, 64, 32)]:
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
    y = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    w = torch.randn(27 * ci * co, device='cuda') * 0.02
    b = torch.zeros(co, device='cuda')
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device='cuda')
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())
    res = {}
    for key in [(0, 0)] + [(mb, acc) for mb in (1, 2, 3, 4, 5) for acc in (1, 2, 3)]:
        lib.vm_debug_set_fwd_plan(*key)
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                def run():
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
            res[key] = e0.elapsed_time(e1) * 1e3 / 50
        except Exception:
            pass
    lib.vm_debug_set_fwd_plan(0, 0)
    best = min((v, k) for k, v in res.items() if k != (0, 0))
    print(f"{ci}->{co} @{e}^3: auto {res[(0, 0)]:.1f} us, best forced {best[0]:.1f} us at (MB, nacc) = {best[1]}; "
          + " ".join(f"{k[0]}/{k[1]}:{v:.1f}" for k, v in sorted(res.items()) if k != (0, 0)))
