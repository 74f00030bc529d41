"""Time every feasible wgrad plan for the cfg2 layer shapes (tuning aid)."""
import ctypes, sys, torch
sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.step import Slab
lib = _lib.load()
names = "runs KS MT mpu ngrp stages ksplit spk units ones stage_bytes gdelta".split()
shapes = [(16, 16, 128), (48, 16, 128), (1, 16, 128), (32, 32, 64), (96, 32, 64), (16, 32, 64), (64, 64, 32),
          (192, 64, 32), (128, 128, 16), (64, 128, 16)]
for cin, cout, e in shapes:
    x = Slab(1, cin, e, e, e, torch.bfloat16, "cuda"); g = Slab(1, cout, e, e, e, torch.bfloat16, "cuda")
    x.storage.normal_(); g.storage.normal_()
    gw = torch.zeros(27 * cin * cout, device="cuda"); gb = torch.zeros(cout, device="cuda")
    res = []
    for fold in (0,):  # (the kw-folded variant was removed; kept as a 1-element loop)
      for runs in (0, 1):
          for ks in (64, 128, 192, 256):
              for mpu in range(1, 10):
                  lib.vm_debug_force_wgrad_plan(runs, ks, mpu)
                  out = (ctypes.c_int * 12)()
                  if lib.vm_debug_wgrad_plan(1, cin, cout, e, e, e, out) != 0:
                      continue
                  pl = dict(zip(names, list(out)))
                  if pl["runs"] != runs or pl["KS"] != ks or pl["mpu"] != mpu:
                      continue
                  nb = lib.vm_conv3d_wgrad_tc_ws(1, cin, cout, e, e, e)
                  ws = torch.empty(nb // 4 + 64, device="cuda")
                  st = _lib.stream_ptr()
                  args = (x.p(), x.bstride, g.p(), g.bstride, _lib.ptr(gw), _lib.ptr(gb), _lib.ptr(ws), 1, cin, cout, e, e, e, st)
                  _lib.call("vm_conv3d_wgrad_tc", *args)
                  e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                  e0.record()
                  for _ in range(5):
                      _lib.call("vm_conv3d_wgrad_tc", *args)
                  e1.record(); torch.cuda.synchronize()
                  res.append((round(e0.elapsed_time(e1) / 5 * 1e3, 1), "fold%d" % fold, runs, ks, mpu, pl["stages"]))
    lib.vm_debug_force_wgrad_plan(-1, 0, 0)
    out = (ctypes.c_int * 12)(); lib.vm_debug_wgrad_plan(1, cin, cout, e, e, e, out)
    pl = dict(zip(names, list(out)))
    res.sort()
    print(f"{cin:4d}->{cout:4d} @{e:4d}: best {res[0]}  | model picks runs={pl['runs']} KS={pl['KS']} mpu={pl['mpu']} | top5 {res[:5]}", flush=True)
