"""A/B of the kw-stacked sweep (Nc = 16) plans: MB and segment length forced."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
ci, co, e = 16, 16, 128
x = Slab(1, ci, e, e, e, torch.bfloat16, "cuda")
x.storage.normal_()
y = Slab(1, co, e, e, e, torch.bfloat16, "cuda")
w = torch.randn(27 * ci * co, device="cuda") * 0.05
b = torch.zeros(co, device="cuda")
wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device="cuda")
_lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())


def run():
    _lib.call("vm_conv3d_fwd_tc", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride, None, 0, 1, ci, co,
              e, e, e, 1, _lib.stream_ptr())


for mb in (1, 2):
    for s in (0, 8, 16, 32, 64, 128):
        lib.vm_debug_set_sweep_mb(mb)
        lib.vm_debug_set_sweep_s(s)
        try:
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                run()
            e1.record()
            torch.cuda.synchronize()
            print(f"MB={mb} S={s}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
        except Exception as ex:  # noqa: BLE001
            print(f"MB={mb} S={s}: {ex}")
lib.vm_debug_set_sweep_mb(0)
lib.vm_debug_set_sweep_s(0)
