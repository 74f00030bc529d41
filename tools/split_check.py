import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.step import Slab
lib = _lib.load()
for (ci, co, d, e) in [(768, 256, 4, 32), (512, 512, 2, 16), (128, 128, 16, 16)]:
    x = Slab(1, ci, d, e, e, torch.bfloat16, "cuda"); x.storage.normal_()
    y = Slab(1, co, d, e, e, torch.bfloat16, "cuda")
    w = torch.randn(27 * ci * co, device="cuda") * 0.05
    b = torch.zeros(co, device="cuda")
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())
    nb = _lib.call_size("vm_conv3d_fwd_tc_ws_bytes", 1, ci, co, d, e, e)
    ws = torch.zeros(max(nb, 16) // 4 + 64, device="cuda")
    outs = {}
    for ms in (1, 2, 4, 8, 12):
        lib.vm_debug_set_fwd_plan(1, 1); lib.vm_debug_set_fwd_max_split(16); lib.vm_debug_force_fwd_split(ms)
        rs = []
        for rep in range(3):
            y.storage.zero_()
            try:
                _lib.call("vm_conv3d_fwd_tc_ws", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride, None, 0,
                          1, ci, co, d, e, e, 1, _lib.ptr(ws), nb, _lib.stream_ptr())
            except Exception as ex:
                rs = None; break
            torch.cuda.synchronize(); rs.append(y.storage.float().clone())
        if rs is None: continue
        det = all(torch.equal(rs[0], r) for r in rs[1:])
        outs[ms] = rs[0]
        base = outs[min(outs)]
        rel = float((rs[0] - base).norm() / base.norm())
        print(f"{ci}->{co} @{d}x{e}^2 split {ms}: deterministic={det} rel-vs-split1={rel:.2e}", flush=True)
    lib.vm_debug_set_fwd_plan(0, 0); lib.vm_debug_force_fwd_split(0)
