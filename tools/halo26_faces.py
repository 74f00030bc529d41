"""Loopback time (pack + device copy + unpack, no NCCL) of vm_halo_slab_fwd26 restricted to the
D, H or W face pair, the 12 edges, or all 26 directions, on one slab (C:E args)."""
import ctypes
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.halo import directions26, nccl_comm_ptr  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

with socket.socket() as s_:
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
comm = nccl_comm_ptr()
lib = _lib.load()
lib.vm_debug_halo_loopback(1)
dirs = directions26()
sel = {"D": lambda s: s[1] == 0 and s[2] == 0, "H": lambda s: s[0] == 0 and s[2] == 0,
       "W": lambda s: s[0] == 0 and s[1] == 0, "edges": lambda s: sum(v != 0 for v in s) == 2,
       "all": lambda s: True}
for spec in sys.argv[1:] or ["32:256"]:
    C, E = (int(v) for v in spec.split(":"))
    sl = Slab(1, C, E, E, E, torch.bfloat16, "cuda")
    sl.storage.normal_()
    wsb = _lib.call_size("vm_halo_slab_ws_bytes26", _lib.VM_BF16, 1, C, E, E, E)
    ws = torch.empty(wsb // 4 + 64, device="cuda")
    out = []
    for name, f in sel.items():
        n26 = [0 if f(s) else -1 for s in dirs]

        def call():
            _lib.call("vm_halo_slab_fwd26", ctypes.c_void_p(comm), _lib.VM_BF16, sl.p(), sl.bstride, 1, C, E, E, E,
                      (ctypes.c_int * 26)(*n26), _lib.ptr(ws), ws.numel() * 4, None, _lib.stream_ptr())

        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            call()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(10):
                    call()
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            e1.synchronize()
        out.append(f"{name} {e0.elapsed_time(e1) / 10 * 1e3:.1f}")
    print(f"C={C} E={E} loopback us: " + ", ".join(out), flush=True)
lib.vm_debug_halo_loopback(0)
dist.destroy_process_group()
