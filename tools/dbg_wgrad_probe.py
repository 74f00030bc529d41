"""Cycle probes of the kd-along-N weight-gradient kernel (vm_debug_set_fwd_probe)."""
import ctypes
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
buf = torch.zeros(148 * 8, dtype=torch.int64, device='cuda')
lib.vm_debug_set_fwd_probe.argtypes = [ctypes.c_void_p]
for (ci, co, e) in [(16, 16, 128), (48, 16, 128), (32, 32, 64)]:
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
    g = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device='cuda')
    gb = torch.zeros(co, device='cuda')
    ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device='cuda')
    st = _lib.stream_ptr()
    for it in range(3):
        buf.zero_()
        lib.vm_debug_set_fwd_probe(ctypes.c_void_p(buf.data_ptr()) if it == 2 else None)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb), _lib.ptr(ws),
                  1, ci, co, e, e, e, st)
        e1.record()
        torch.cuda.synchronize()
    lib.vm_debug_set_fwd_probe(None)
    d = buf.view(148, 8).cpu().float()
    act = d[d[:, 0] > 0]
    m = act.mean(0).tolist()
    print(f"{ci}->{co} @{e}^3 {e0.elapsed_time(e1) * 1e3:.1f}us ctas={len(act)} | MMA total {m[0]:.0f} "
          f"wait_full {m[2]:.0f} issue {m[3]:.0f} | PROD wait_empty {m[7]:.0f}")
