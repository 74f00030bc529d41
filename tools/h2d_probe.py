import torch, time
x = torch.empty(8*1024*1024//4*4, dtype=torch.float32).pin_memory()
d = torch.empty_like(x, device='cuda')
s = torch.cuda.Stream()
for it in range(3):
    ts=[]
    for k in range(20):
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); d.copy_(x, non_blocking=True); e1.record(s)
        e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print("H2D 32MB ms: min %.3f max %.3f" % (min(ts), max(ts)), "GB/s %.1f" % (x.numel()*4/min(ts)/1e6))
