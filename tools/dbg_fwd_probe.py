"""Cycle probes of the general forward kernel (k_conv_fwd_tc, vm_debug_set_fwd_probe) with the
split-K limit 1 and 3 (vm_debug_set_fwd_max_split): per-CTA MMA loop, waits, epilogue total
and the last split's fix-up."""
import ctypes
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
buf = torch.zeros(148 * 8, dtype=torch.int64, device='cuda')
lib.vm_debug_set_fwd_probe.argtypes = [ctypes.c_void_p]
SHAPES = [tuple(int(v) for v in a.split(':')) for a in sys.argv[1:]] or [(64, 64, 32, 32), (128, 128, 16, 16), (64, 128, 16, 16), (192, 64, 32, 32)]
for (ci, co, e, dd) in SHAPES:
    x = Slab(1, ci, dd, e, e, torch.bfloat16, 'cuda')
    y = Slab(1, co, dd, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    w = torch.randn(27 * ci * co, device='cuda') * 0.05
    b = torch.zeros(co, device='cuda')
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device='cuda')
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())
    nb = _lib.call_size("vm_conv3d_fwd_tc_ws_bytes", 1, ci, co, dd, e, e)
    ws = torch.zeros(max(nb, 16) // 4 + 64, device='cuda')
    for ms, fl in ((1, 1), (1, 1 | (1 << 9)), (1, 1 | (1 << 11)), (2, 1)):
        lib.vm_debug_force_fwd_split(ms)
        for it in range(3):
            buf.zero_()
            lib.vm_debug_set_fwd_probe(ctypes.c_void_p(buf.data_ptr()) if it == 2 else None)
            _lib.call("vm_conv3d_fwd_tc_ws", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride, None, 0,
                      1, ci, co, dd, e, e, fl, _lib.ptr(ws), nb, _lib.stream_ptr())
            torch.cuda.synchronize()
        lib.vm_debug_set_fwd_probe(None)
        d = buf.view(148, 8).cpu().float()
        act = d[d[:, 0] > 0]
        m = act.mean(0).tolist()
        mx = act.max(0).values.tolist()
        print(f"{ci}->{co} @{dd}x{e}^2 split={ms} flags {fl:#x}: ctas={len(act)} MMA loop {m[0]:.0f} (max {mx[0]:.0f}) "
              f"wait_tmem {m[1]:.0f} wait_full {m[2]:.0f} | epi total {m[4]:.0f} (max {mx[4]:.0f}) "
              f"epi_wait {m[3]:.0f} fixup {m[5]:.0f} (max {mx[5]:.0f}) drain|publish {m[6]:.0f} (max {mx[6]:.0f}) "
              f"epi-start|arrive {m[7]:.0f} (max {mx[7]:.0f})")
    lib.vm_debug_force_fwd_split(0)
