"""Device time of one peer-memory depth push (vm_halo_depth_push, self neighbours) per slab
shape, replayed in a CUDA graph: python tools/push_time.py C:D:H:W ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_03108_b200.halo import PeerDepthHalo  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

from paper_1909_03108_b200 import _lib  # noqa: E402

specs = [a for a in sys.argv[1:] if ":" in a]
mode = int(os.environ.get("PUSH_MODE", "0"))
_lib.load().vm_debug_push_mode(mode)
print("mode", mode)
for spec in specs:
    C, D, H, W = (int(v) for v in spec.split(":"))
    s = Slab(1, C, D, H, W, torch.bfloat16, "cuda")
    halo = PeerDepthHalo([0, 0, -1, -1, -1, -1], "cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        halo.begin_step()
        halo.forward(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            halo.begin_step()
            for _ in range(20):
                halo.forward(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 100 * 1e3
    layer = (H + 2) * (W + 2) * ((C + 7) // 8) * 16
    print(f"C={C:4d} D={D:3d} {H}x{W}: {us:7.2f} us per push, {2 * 2 * layer / us / 1e3:7.1f} GB/s (read+write)")
    halo.check()
