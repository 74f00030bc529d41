"""Cycle probes of the kd-stacked sweep conv kernel (vm_debug_set_fwd_probe)."""
import ctypes
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
buf = torch.zeros(148 * 8, dtype=torch.int64, device='cuda')
lib.vm_debug_set_fwd_probe.argtypes = [ctypes.c_void_p]
lib.vm_debug_set_sweep_mode.argtypes = [ctypes.c_int]
MODES = [int(v) for v in sys.argv[1:]] or [0]
for (ci, co, e, mode) in [(ci, co, e, m) for m in MODES for (ci, co, e) in [(16, 16, 128), (48, 16, 128), (32, 32, 64), (16, 32, 64)]] + [(16, 16, 128, 'dgrad'), (32, 32, 64, 'dgrad')]:
    dgrad = mode == 'dgrad'
    lib.vm_debug_set_sweep_mode(0 if dgrad else mode)
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
    y = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    w = torch.randn(27 * ci * co, device='cuda') * 0.05
    b = torch.zeros(co, device='cuda')
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device='cuda')
    st = _lib.stream_ptr()
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, st)
    for it in range(3):
        buf.zero_()
        lib.vm_debug_set_fwd_probe(ctypes.c_void_p(buf.data_ptr()) if it == 2 else None)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if dgrad:  # masked, no bias (the dgrad epilogue)
            _lib.call("vm_conv3d_fwd_tc", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride, y.p(),
                      y.bstride, 1, ci, co, e, e, e, 2 | 4, st)
        else:
            _lib.call("vm_conv3d_fwd_tc", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride, None, 0, 1,
                      ci, co, e, e, e, 1, st)
        e1.record()
        torch.cuda.synchronize()
    lib.vm_debug_set_fwd_probe(None)
    d = buf.view(148, 8).cpu().float()
    act = d[d[:, 0] > 0]
    m = act.mean(0).tolist()
    print(f"mode {mode} {ci}->{co} @{e}^3 {e0.elapsed_time(e1) * 1e3:.1f}us ctas={len(act)} | MMA total {m[0]:.0f} "
          f"wait_tempty {m[1]:.0f} wait_full {m[2]:.0f} issue {m[3]:.0f} | EPI total {m[4]:.0f} wait {m[5]:.0f} "
          f"seqs {m[6]:.0f} | PROD wait_empty {m[7]:.0f}")
