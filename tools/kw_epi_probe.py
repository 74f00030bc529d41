"""Epilogue sub-phase cycle probes of k_conv_fwd_sweepkw (DBG variant)."""
import ctypes, sys
import torch
sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.step import Slab
lib = _lib.load()
buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
lib.vm_debug_set_fwd_probe.argtypes = [ctypes.c_void_p]
for ci, co, e in [(16, 16, 128), (48, 16, 128)]:
    x = Slab(1, ci, e, e, e, torch.bfloat16, "cuda"); x.storage.normal_()
    y = Slab(1, co, e, e, e, torch.bfloat16, "cuda")
    w = torch.randn(27 * ci * co, device="cuda") * 0.05
    b = torch.zeros(co, device="cuda")
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())
    lib.vm_debug_set_fwd_probe(ctypes.c_void_p(buf.data_ptr()))
    _lib.call("vm_conv3d_fwd_tc", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride, None, 0, 1, ci, co, e, e, e, 1, _lib.stream_ptr())
    torch.cuda.synchronize()
    lib.vm_debug_set_fwd_probe(None)
    d = buf.view(148, 8).cpu().float()
    act = d[d[:, 4] > 0]
    m = act.mean(0).tolist()
    print(f"{ci}->{co}: EPI total {m[4]:.0f} wait {m[5]:.0f} blocks {m[6]:.0f} | ld {m[7]:.0f} xch {m[1]:.0f} math+xch {m[2]:.0f} stwait {m[3]:.0f}")
