import ctypes, torch, sys, os
sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.step import Slab
lib=_lib.load()
buf=torch.zeros(148*8, dtype=torch.int64, device='cuda')
lib.vm_debug_set_fwd_probe.argtypes=[ctypes.c_void_p]
SHAPES=[(64,64,32),(128,128,16),(64,128,16),(192,64,32),(96,32,64)]
for (ci,co,e,fl) in [(ci,co,e,1) for (ci,co,e) in SHAPES]:
    x=Slab(1,ci,e,e,e,torch.bfloat16,'cuda'); y=Slab(1,co,e,e,e,torch.bfloat16,'cuda'); x.storage.normal_()
    w=torch.randn(27*ci*co,device='cuda')*0.05; b=torch.zeros(co,device='cuda')
    wp=torch.empty(_lib.call_size("vm_packed_weights_bytes",ci,co)//2,dtype=torch.bfloat16,device='cuda')
    st=_lib.stream_ptr()
    _lib.call("vm_pack_weights",_lib.ptr(w),_lib.ptr(wp),ci,co,0,st)
    for it in range(3):
        buf.zero_()
        lib.vm_debug_set_fwd_probe(ctypes.c_void_p(buf.data_ptr()) if it==2 else None)
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("vm_conv3d_fwd_tc",x.p(),x.bstride,_lib.ptr(wp),_lib.ptr(b),y.p(),y.bstride,None,0,1,ci,co,e,e,e,fl,st)
        e1.record(); torch.cuda.synchronize()
    d=buf.view(2,148,4).cpu().float()
    act=d[0][d[0][:,0]>0]
    print(hex(fl), ci,co,e, f"{e0.elapsed_time(e1)*1e3:.1f}us ctas={len(act)}", "MMA: total %.0f wait_tmem %.0f wait_full %.0f epi_wait %.0f" % tuple(act.mean(0).tolist()))
