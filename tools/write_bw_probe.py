import torch
x = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
y = torch.empty(1 << 27, dtype=torch.bfloat16, device="cuda")
for name, fn, nbytes in (("fill 2GB", lambda: x.fill_(1.0), 2 << 30), ("zero 2GB", lambda: x.zero_(), 2 << 30),
                         ("copy 256MB->2GB? (repeat)", lambda: x.view(8, -1).copy_(y.view(1, -1).expand(8, -1)), (2 << 30) + (256 << 20))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): fn()
    e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"{name}: {t*1e3:.0f} us, {nbytes / t / 1e6:.0f} GB/s")
