"""In-graph time of the general forward kernel per deep-level shape with split-K limited to
1/2/3 (vm_debug_set_fwd_max_split), plus the plan the cost model picks (max 3)."""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
SHAPES = [(32, 64, 32), (64, 64, 32), (192, 64, 32), (64, 128, 16), (128, 128, 16), (128, 64, 32), (96, 32, 64),
          (32, 96, 64), (64, 32, 32), (128, 64, 16)]
for (ci, co, e) in SHAPES:
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
    y = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    w = torch.randn(27 * ci * co, device='cuda') * 0.02
    b = torch.zeros(co, device='cuda')
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device='cuda')
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())
    nb = _lib.call_size("vm_conv3d_fwd_tc_ws_bytes", 1, ci, co, e, e, e)
    ws = torch.zeros(max(nb, 16) // 4 + 64, device='cuda')
    res = []
    for ms in (1, 2, 3):
        lib.vm_debug_set_fwd_max_split(ms)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            def run():
                _lib.call("vm_conv3d_fwd_tc_ws", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride,
                          None, 0, 1, ci, co, e, e, e, 1, _lib.ptr(ws), nb, _lib.stream_ptr())
            run()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
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
        res.append(e0.elapsed_time(e1) * 1e3 / 100)
    lib.vm_debug_set_fwd_max_split(3)
    print(f"{ci}->{co} @{e}^3: max_split 1/2/3 = " + " / ".join(f"{t:.1f}" for t in res) + " us")
