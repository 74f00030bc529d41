"""In-graph cost per launch of a chain of dependent conv launches, with and without
programmatic dependent launch (vm_set_pdl).  Chains x -> y -> x ... (Cin == Cout)."""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
SHAPES = [(128, 128, 16), (64, 64, 32), (32, 32, 64), (16, 16, 128)]
NCH = 20
for (c, _, e) in SHAPES:
    a = Slab(1, c, e, e, e, torch.bfloat16, 'cuda')
    b = Slab(1, c, e, e, e, torch.bfloat16, 'cuda')
    a.storage.normal_()
    w = torch.randn(27 * c * c, device='cuda') * 0.02
    bias = torch.zeros(c, device='cuda')
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", c, c) // 2, dtype=torch.bfloat16, device='cuda')
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), c, c, 0, _lib.stream_ptr())
    res = {}
    outs = {}
    for pdl in (0, 1, 0, 1):
        lib.vm_set_pdl(pdl)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            def chain():
                st = _lib.stream_ptr()
                src, dst = a, b
                for _ in range(NCH):
                    _lib.call("vm_conv3d_fwd_tc", src.p(), src.bstride, _lib.ptr(wp), _lib.ptr(bias), dst.p(),
                              dst.bstride, None, 0, 1, c, c, e, e, e, 1, st)
                    src, dst = dst, src
            chain()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                chain()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[pdl] = e0.elapsed_time(e1) * 1e3 / (10 * NCH)
        outs[pdl] = b.storage.clone()
    same = torch.equal(outs[0], outs[1])
    print(f"conv {c}->{c} @{e}^3: {res[0]:.1f} us/launch plain, {res[1]:.1f} us/launch pdl, bitwise same: {same}")
