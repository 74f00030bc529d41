"""General fwd split-K: determinism, agreement with the unsplit plan, and the cluster (DSMEM)
fix-up bitwise equal to the global-workspace fix-up, at forced splits; in-graph times of each."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
SHAPES = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(128, 128, 16, 16), (64, 128, 16, 16),
                                                                          (512, 512, 2, 16), (768, 256, 4, 32)]


def timed(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (ci, co, d, e) in SHAPES:
    x = Slab(1, ci, d, e, e, torch.bfloat16, "cuda")
    x.storage.normal_()
    y = Slab(1, co, d, e, e, torch.bfloat16, "cuda")
    w = torch.randn(27 * ci * co, device="cuda") * 0.05
    b = torch.randn(co, device="cuda") * 0.1
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", ci, co) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, 0, _lib.stream_ptr())
    nb = _lib.call_size("vm_conv3d_fwd_tc_ws_bytes", 1, ci, co, d, e, e)
    ws = torch.zeros(max(nb, 16) // 4 + 64, device="cuda")

    def run():
        _lib.call("vm_conv3d_fwd_tc_ws", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride, None, 0,
                  1, ci, co, d, e, e, 1, _lib.ptr(ws), nb, _lib.stream_ptr())

    lib.vm_debug_set_fwd_max_split(16)
    lib.vm_debug_force_fwd_split(0)
    lib.vm_debug_set_fwd_cluster(0)
    t_auto = timed(run)
    outs = {}
    line = []
    for ms in (1, 2, 3, 4, 6, 8):
        for cl in (1, 0):
            lib.vm_debug_set_fwd_plan(1, 1)
            lib.vm_debug_force_fwd_split(ms)
            lib.vm_debug_set_fwd_cluster(cl)
            rs = []
            try:
                for _ in range(3):
                    y.storage.zero_()
                    run()
                    torch.cuda.synchronize()
                    rs.append(y.storage.clone())
                t = timed(run)
            except Exception:  # noqa: BLE001
                continue
            det = all(torch.equal(rs[0], r) for r in rs[1:])
            outs[(ms, cl)] = rs[0]
            line.append(f"s{ms}{'c' if cl else 'g'} {t:.1f}{'' if det else ' NONDET'}")
    lib.vm_debug_set_fwd_plan(0, 0)
    lib.vm_debug_force_fwd_split(0)
    lib.vm_debug_set_fwd_cluster(0)
    same = all(torch.equal(outs[(ms, 1)], outs[(ms, 0)]) for ms in (2, 3, 4, 6, 8) if (ms, 1) in outs and (ms, 0) in outs)
    base = outs[(1, 1)].float()
    worst = max(float((o.float() - base).norm() / base.norm()) for o in outs.values())
    print(f"{ci}->{co} @{d}x{e}^2: planner {t_auto:.1f} us | " + ", ".join(line)
          + f" | cluster==global bitwise: {same}, max rel vs unsplit {worst:.1e}", flush=True)
