import sys, torch
sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.step import Slab
lib = _lib.load()
for (ci, co, e) in [(64, 64, 128), (32, 64, 128), (64, 64, 64), (192, 64, 128), (16, 80, 64), (32, 32, 256)]:
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda'); x.storage.normal_()
    g = Slab(1, co, e, e, e, torch.bfloat16, 'cuda'); g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device='cuda'); gb = torch.zeros(co, device='cuda')
    res = {}
    for mode in ("kd", "tc_copies", "tc_auto"):
        if mode == "kd": lib.vm_debug_force_wgrad_plan(-1, 0, 0)
        elif mode == "tc_copies": lib.vm_debug_force_wgrad_plan(0, 0, 0)
        else: lib.vm_debug_force_wgrad_plan(2, 0, 0)  # general kernel, its own staging choice
        try:
            ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device='cuda')
            def run():
                _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb), _lib.ptr(ws), 1, ci, co, e, e, e, _lib.stream_ptr())
            run(); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): run()
            e1.record(); torch.cuda.synchronize()
            res[mode] = e0.elapsed_time(e1) / 5
        except Exception as ex:
            res[mode] = str(ex)[:60]
    lib.vm_debug_force_wgrad_plan(-1, 0, 0)
    print(ci, co, e, res)
    del x, g, ws
    torch.cuda.empty_cache()
