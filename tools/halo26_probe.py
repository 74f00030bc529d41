"""Per-exchange device time of the NCCL slab halo on one GPU (1-rank communicator, every
neighbour = this rank): 3-phase vm_halo_slab_fwd vs one-phase vm_halo_slab_fwd26, each with
NCCL and with the loopback probe (device copies instead of NCCL: pack + unpack cost alone).

usage: python tools/halo26_probe.py [C:E ...]   (channels : cubic local extent)"""
import ctypes
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.halo import nbr26_of, nccl_comm_ptr  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

with socket.socket() as s_:
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
comm = nccl_comm_ptr()
lib = _lib.load()
shapes = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(32, 256), (64, 128), (128, 64), (512, 16), (1024, 8)]
nbr6 = [0] * 6
n26 = nbr26_of(nbr6)
for C, E in shapes:
    s = Slab(1, C, E, E, E, torch.bfloat16, "cuda")
    s.storage.normal_()
    res = {}
    for name, fn26 in (("3-phase", False), ("1-phase", True)):
        wsb = _lib.call_size("vm_halo_slab_ws_bytes26" if fn26 else "vm_halo_slab_ws_bytes", _lib.VM_BF16, 1, C, E, E, E)
        ws = torch.empty(wsb // 4 + 64, device="cuda")

        def call():
            if fn26:
                _lib.call("vm_halo_slab_fwd26", ctypes.c_void_p(comm), _lib.VM_BF16, s.p(), s.bstride, 1, C, E, E, E,
                          (ctypes.c_int * 26)(*n26), _lib.ptr(ws), ws.numel() * 4, None, _lib.stream_ptr())
            else:
                _lib.call("vm_halo_slab_fwd", ctypes.c_void_p(comm), _lib.VM_BF16, s.p(), s.bstride, 1, C, E, E, E,
                          (ctypes.c_int * 6)(*nbr6), _lib.ptr(ws), ws.numel() * 4, None, _lib.stream_ptr())

        for lb in (0, 1):
            lib.vm_debug_halo_loopback(lb)
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                call()
                torch.cuda.synchronize()
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
            res[f"{name}{' loopback' if lb else ''}"] = e0.elapsed_time(e1) / 10 * 1e3
        lib.vm_debug_halo_loopback(0)
    print(f"C={C} E={E}: " + ", ".join(f"{k} {v:.1f} us" for k, v in res.items()), flush=True)
dist.destroy_process_group()
