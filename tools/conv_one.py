"""Run one conv kernel (fwd | dgrad | wgrad) of a given shape a few times — the target of
single-kernel ncu captures:  python tools/conv_one.py fwd 128 128 16 [reps]."""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

kind, ci, co, e = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
st = _lib.stream_ptr()
x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
x.storage.normal_()
if kind in ("fwd", "dgrad"):
    cin, cout = (ci, co) if kind == "fwd" else (co, ci)
    y = Slab(1, cout, e, e, e, torch.bfloat16, 'cuda')
    w = torch.randn(27 * ci * co, device='cuda') * 0.05
    b = torch.zeros(cout, device='cuda')
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", cin, cout) // 2, dtype=torch.bfloat16, device='cuda')
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, int(kind == "dgrad"), st)
    src = x if kind == "fwd" else Slab(1, cin, e, e, e, torch.bfloat16, 'cuda')
    src.storage.normal_()
    flags = 1 if kind == "fwd" else 2 | 4
    m = y if kind == "dgrad" else None
    for _ in range(reps):
        _lib.call("vm_conv3d_fwd_tc", src.p(), src.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride,
                  m.p() if m is not None else None, m.bstride if m is not None else 0, 1, cin, cout, e, e, e, flags, st)
else:
    g = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device='cuda')
    gb = torch.zeros(co, device='cuda')
    ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device='cuda')
    for _ in range(reps):
        _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb), _lib.ptr(ws),
                  1, ci, co, e, e, e, st)
torch.cuda.synchronize()
print("ok", kind, ci, co, e)
