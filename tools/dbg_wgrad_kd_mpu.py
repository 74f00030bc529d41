import sys, torch
sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.step import Slab
lib = _lib.load()
for (ci, co, e) in [(48, 16, 128), (96, 32, 64), (48, 32, 64)]:
    x = Slab(1, ci, e, e, e, torch.bfloat16, 'cuda'); x.storage.normal_()
    g = Slab(1, co, e, e, e, torch.bfloat16, 'cuda'); g.storage.normal_()
    gw = torch.zeros(27 * ci * co, device='cuda'); gb = torch.zeros(co, device='cuda')
    res = {}
    for mpu in (0, 1, 2, 3):
        lib.vm_debug_force_wgrad_plan(-1, 0, mpu)
        ws = torch.empty(_lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, e, e, e) // 4 + 64, device='cuda')
        def run():
            _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb), _lib.ptr(ws), 1, ci, co, e, e, e, _lib.stream_ptr())
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            run(); torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(10): run()
        gr.replay(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): gr.replay()
        e1.record(); torch.cuda.synchronize()
        res[mpu] = round(e0.elapsed_time(e1) * 1e3 / 50, 1)
    lib.vm_debug_force_wgrad_plan(-1, 0, 0)
    print(ci, co, e, res)
