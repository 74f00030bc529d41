import ctypes, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1909_03108_b200 import _lib
from tests.test_gpu_conv import _slab_from, _wgrad
from oracle import voxmesh_oracle as O
lib = _lib.load()
names = "runs KS MT mpu ngrp stages ksplit spk units ones stage_bytes gdelta".split()
for shape in [(1, 32, 32, 6, 8, 64), (1, 16, 16, 4, 8, 128), (1, 16, 16, 128, 128, 128), (1, 48, 16, 128, 128, 128),
              (1, 32, 32, 64, 64, 64), (1, 64, 32, 64, 64, 64), (1, 64, 64, 32, 32, 32)]:
    B, cin, cout, D, H, W = shape
    out = (ctypes.c_int * 12)()
    lib.vm_debug_wgrad_plan(B, cin, cout, D, H, W, out)
    print(shape, dict(zip(names, list(out))))
    if D > 8:
        continue
    rng = np.random.default_rng(1)
    x = O.bf16_round(rng.standard_normal((B, D, H, W, cin)).astype(np.float32))
    g = O.bf16_round(rng.standard_normal((B, D, H, W, cout)).astype(np.float32))
    xs, gs = _slab_from(x), _slab_from(g)
    gw, gb = _wgrad("vm_conv3d_wgrad_tc", xs, gs, cin, cout)
    sw, sb = _wgrad("vm_conv3d_wgrad_simt", xs, gs, cin, cout)
    bad = np.abs(gw - sw) > 1e-3 * np.abs(sw).max()
    idx = np.argwhere(bad)
    print("  bad", bad.sum(), "of", bad.size, "bias err", np.abs(gb - sb).max())
    if len(idx):
        t = idx[:, 0] * 9 + idx[:, 1] * 3 + idx[:, 2]
        print("  taps", np.unique(t), "ci", np.unique(idx[:, 3]), "co", np.unique(idx[:, 4])[:40])
