"""Run the Cin = 1 first-layer kernels once per rep at 128^3 (ncu target)."""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "fwd"
e, co = 128, 16
xd = torch.randn(e, e, e, device='cuda')
x1 = torch.empty((e + 2) ** 3, dtype=torch.bfloat16, device='cuda')
_lib.call("vm_dense_to_compact1", _lib.ptr(xd), _lib.ptr(x1), 1, e, e, e, _lib.stream_ptr())
w = torch.randn(27 * co, device='cuda') * 0.1
b = torch.zeros(co, device='cuda')
y = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
y.storage.normal_()
gw = torch.zeros(27 * co, device='cuda')
gb = torch.zeros(co, device='cuda')
ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_c1_ws", 1, co, e, e, e) // 4 + 64, device='cuda')
for _ in range(3):
    if kind == "fwd":
        _lib.call("vm_conv3d_fwd_c1", _lib.ptr(x1), 0, _lib.ptr(w), _lib.ptr(b), y.p(), y.bstride, 1, co, e, e, e, 1,
                  _lib.stream_ptr())
    else:
        _lib.call("vm_conv3d_wgrad_c1", _lib.ptr(x1), 0, y.p(), y.bstride, _lib.ptr(gw), _lib.ptr(gb), _lib.ptr(ws),
                  1, co, e, e, e, _lib.stream_ptr())
torch.cuda.synchronize()
print("ok", kind)
