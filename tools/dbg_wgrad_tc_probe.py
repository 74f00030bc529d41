"""Cycle probes + in-graph time of the general weight-gradient kernel (k_conv_wgrad_tc) at
the deep-level shapes (vm_debug_set_fwd_probe; plan from vm_debug_wgrad_plan)."""
import ctypes
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.step import Slab  # noqa: E402

lib = _lib.load()
buf = torch.zeros(148 * 8, dtype=torch.int64, device='cuda')
lib.vm_debug_set_fwd_probe.argtypes = [ctypes.c_void_p]
SHAPES = [(64, 64, 32), (192, 64, 32), (128, 128, 16), (64, 128, 16), (32, 64, 32)]
MIN_SPK = [2]
args = sys.argv[1:]
FORCE = None
if args and args[0].startswith('force='):  # force=runs,ks,mpu
    FORCE = [int(v) for v in args.pop(0)[6:].split(',')]
    lib.vm_debug_force_wgrad_plan(*FORCE)
if args and args[0].startswith('spk='):
    MIN_SPK = [int(v) for v in args.pop(0)[4:].split(',')]
if args:
    SHAPES = [tuple(int(v) for v in a.split(',')) for a in args]
SHAPES = [(ci, co, e, spk) for spk in MIN_SPK for (ci, co, e) in SHAPES]
for (ci, co, e, spk) in SHAPES:
    lib.vm_debug_set_wgrad_min_spk(spk)
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda')
    g = Slab(1, co, e, e, e, torch.bfloat16, 'cuda')
    x.storage.normal_()
    g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device='cuda')
    gb = torch.zeros(co, device='cuda')
    ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device='cuda')
    plan = (ctypes.c_int * 12)()
    lib.vm_debug_wgrad_plan(1, ci, co, e, e, e, plan)
    st = _lib.stream_ptr()

    def run():
        _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb),
                  _lib.ptr(ws), 1, ci, co, e, e, e, _lib.stream_ptr())
    run()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        run()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(10):
                run()
    gr.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) * 1e3 / 50
    buf.zero_()
    lib.vm_debug_set_fwd_probe(ctypes.c_void_p(buf.data_ptr()))
    run()
    torch.cuda.synchronize()
    lib.vm_debug_set_fwd_probe(None)
    d = buf.view(148, 8).cpu().float()
    act = d[d[:, 1] > 0]
    m = act.mean(0).tolist()
    mx = act.max(0).values.tolist()
    names = "runs KS MT mpu ngroups stages ksplit spk units ones stage_bytes gdelta".split()
    print(f"[min_spk {spk}] {ci}->{co} @{e}^3 wgrad+finalize {t_graph:.1f} us/call (graph) ctas={len(act)} plan "
          + " ".join(f"{n}={v}" for n, v in zip(names, plan)))
    print(f"   cycles: setup {m[0]:.0f} | MMA loop {m[1]:.0f} (max {mx[1]:.0f}) first_full {m[2]:.0f} "
          f"wait_full {m[3]:.0f} | epilogue end {m[4]:.0f} (max {mx[4]:.0f}) | PROD wait_empty {m[5]:.0f}")
