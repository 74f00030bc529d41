"""CUDA-event time of one conv kernel call (fwd | dgrad | wgrad) per shape, replayed in a graph.

usage: python tools/conv_time.py wgrad:96:32:256 fwd:16:16:128 ...   (kind:Cin:Cout:extent[:D])
"""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402


def run(kind, ci, co, e, d):
    st = _lib.stream_ptr()
    x = Slab(1, ci, d, e, e, torch.bfloat16, "cuda")
    x.storage.normal_()
    g = Slab(1, co, d, e, e, torch.bfloat16, "cuda")
    g.storage.normal_()
    flops = 2.0 * d * e * e * 27 * ci * co
    if kind in ("fwd", "dgrad"):
        cin, cout = (ci, co) if kind == "fwd" else (co, ci)
        src, dst = (x, Slab(1, co, d, e, e, torch.bfloat16, "cuda")) if kind == "fwd" else (g, Slab(1, ci, d, e, e, torch.bfloat16, "cuda"))
        w = torch.randn(27 * ci * co, device="cuda") * 0.05
        b = torch.zeros(max(ci, co), device="cuda")
        wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", cin, cout) // 2, dtype=torch.bfloat16, device="cuda")
        _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, int(kind == "dgrad"), st)
        mask = x if kind == "dgrad" else None
        flags = (_lib.VM_CONV_MASK | _lib.VM_CONV_NOBIAS) if kind == "dgrad" else _lib.VM_CONV_RELU

        def fn():
            _lib.call("vm_conv3d_fwd_tc", src.p(), src.bstride, _lib.ptr(wp), _lib.ptr(b), dst.p(), dst.bstride,
                      mask.p() if mask else None, mask.bstride if mask else 0, 1, cin, cout, d, e, e, flags,
                      _lib.stream_ptr())
    else:
        gw = torch.zeros(27 * ci * co, device="cuda")
        gb = torch.zeros(co, device="cuda")
        ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, d, e, e) // 4 + 64, device="cuda")

        def fn():
            _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb),
                      _lib.ptr(ws), 1, ci, co, d, e, e, _lib.stream_ptr())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(5):
                fn()
        gr.replay()
        torch.cuda.synchronize()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(4):
            gr.replay()
        b_.record(s)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b_) / 20
    print(f"{kind:5s} {ci:4d}->{co:4d} {d}x{e}x{e}: {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TFLOP/s")


for spec in sys.argv[1:]:
    f = spec.split(":")
    kind, ci, co, e = f[0], int(f[1]), int(f[2]), int(f[3])
    d = int(f[4]) if len(f) > 4 else e
    run(kind, ci, co, e, d)
