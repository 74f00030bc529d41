"""Run one conv layer's kernels (fwd / dgrad / wgrad) on synthetic slabs — for ncu captures.

usage: python tools/kernel_bench.py [fwd|dgrad|wgrad] CIN COUT EXTENT [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402


def main():
    kind = sys.argv[1]
    cin, cout, e = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    B, D, H, W = 1, e, e, e
    x = Slab(B, cin, D, H, W, torch.bfloat16, "cuda")
    g = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
    x.storage.normal_()
    g.storage.normal_()
    st = _lib.stream_ptr()
    w = torch.randn(27 * cin * cout, device="cuda") * 0.05
    b = torch.zeros(max(cin, cout), device="cuda")
    if kind in ("fwd", "dgrad"):
        ci, co = (cin, cout) if kind == "fwd" else (cout, cin)
        src, dst = (x, Slab(B, cout, D, H, W, torch.bfloat16, "cuda")) if kind == "fwd" else (g, Slab(B, cin, D, H, W, torch.bfloat16, "cuda"))
        wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device="cuda")
        _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), cin, cout, int(kind == "dgrad"), st)
        mask = x if kind == "dgrad" else None
        flags = (_lib.VM_CONV_MASK | _lib.VM_CONV_NOBIAS) if kind == "dgrad" else _lib.VM_CONV_RELU
        for _ in range(reps):
            _lib.call("vm_conv3d_fwd_tc", src.p(), src.bstride, _lib.ptr(wp), _lib.ptr(b), dst.p(), dst.bstride,
                      mask.p() if mask else None, mask.bstride if mask else 0, B, ci, co, D, H, W, flags, st)
    else:
        gw = torch.zeros(27 * cin * cout, device="cuda")
        gb = torch.zeros(cout, device="cuda")
        ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", B, cin, cout, D, H, W) // 4 + 64, device="cuda")
        for _ in range(reps):
            _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb),
                      _lib.ptr(ws), B, cin, cout, D, H, W, st)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
