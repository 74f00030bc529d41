"""A/B of the head backward kernels (team kernel vs k_head_bwd_grp): time and output diff.
Args: C:extent ... (bf16, 3 classes)."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
for spec in sys.argv[1:] or ["16:128", "32:256"]:
    C, E = (int(v) for v in spec.split(":"))
    NC = 3
    y = Slab(1, C, E, E, E, torch.bfloat16, "cuda")
    y.storage.normal_()
    gs = Slab(1, C, E, E, E, torch.bfloat16, "cuda")
    w = torch.randn(C * NC, device="cuda") * 0.2
    b = torch.randn(NC, device="cuda") * 0.1
    lab = torch.randint(0, NC, (E * E * E,), dtype=torch.uint8, device="cuda")
    stats = torch.rand(3 * NC + 1, device="cuda") * 1000 + 10
    nb = int(lib.vm_head_partials_count(1, E, E, E))
    wp = torch.zeros(nb * (C * NC + NC), device="cuda")
    res = {}
    for rep in range(3):
        for on in (0, 1):
            lib.vm_debug_set_head_team(on)
            fn = lambda: _lib.call("vm_head_bwd", _lib.VM_BF16, y.p(), y.bstride, _lib.ptr(w), _lib.ptr(b),  # noqa: E731
                                   _lib.ptr(lab), _lib.ptr(stats), gs.p(), gs.bstride, _lib.ptr(wp), 1, C, NC,
                                   E, E, E, 0.9, 0.1, float(E ** 3), 6, 1e-12, 1, _lib.stream_ptr())
            fn()
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                fn()
            e.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(e) / 10 * 1e3
            res[on] = (min(t, res.get(on, (1e9,))[0]), gs.storage.clone(), wp.view(nb, -1).double().sum(0))
    lib.vm_debug_set_head_team(1)
    dg = float((res[0][1].float() - res[1][1].float()).abs().max())
    dw = float((res[0][2] - res[1][2]).norm() / res[0][2].norm())
    nbytes = 2 * (E ** 3) * C * 2 + E ** 3
    print(f"C={C} {E}^3: grp {res[0][0]:.1f} us, team {res[1][0]:.1f} us ({nbytes / res[1][0] / 1e3:.0f} GB/s)"
          f"  max|dg| {dg:.2e}  rel dW {dw:.2e}", flush=True)
