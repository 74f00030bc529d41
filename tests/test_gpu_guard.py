"""Stand-in for compute-sanitizer (closed on this GPU pool: runs under it left GPUs needing a
reset): every tensor-core conv kernel, run on slabs fenced by canary bytes, must (1) leave the
canaries and the output slab's margin shell untouched (no stray stores), and (2) produce
bitwise-identical results over repeated launches (a shared-memory / TMEM / mbarrier race shows
up as run-to-run differences at these shapes: every pipeline stage, ring position and split is
exercised several times)."""

import numpy as np
import pytest
import torch

from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.step import Slab

pytestmark = pytest.mark.gpu

GUARD = 1 << 16  # elements of canary on each side


def _fenced(B, C, D, H, W, fill):
    s = Slab(B, C, D, H, W, torch.bfloat16, "cuda")
    n = s.storage.numel()
    big = torch.full((n + 2 * GUARD,), fill, dtype=torch.bfloat16, device="cuda")
    s.storage = big[GUARD:GUARD + n]
    s.storage.zero_()
    return s, big


def _canaries_ok(big, n, fill):
    v = big.view(torch.int16).cpu().numpy()
    want = np.int16(torch.tensor([fill], dtype=torch.bfloat16).view(torch.int16).item())
    return bool((v[:GUARD] == want).all() and (v[GUARD + n:] == want).all())


def _shell(s):
    v = s.storage[: s.B * s.bstride].view(s.B, s.CG, s.D + 2, s.H + 2, s.W + 2, 8).float().cpu()
    mask = torch.ones_like(v, dtype=torch.bool)
    mask[:, :, 1:-1, 1:-1, 1:-1] = False
    return v[mask]


FWD = [(16, 16, 8, 10, 40), (48, 16, 6, 6, 34), (16, 48, 5, 7, 36), (32, 32, 6, 8, 64), (64, 64, 6, 6, 12),
       (128, 128, 4, 4, 8), (16, 32, 4, 9, 40)]


@pytest.mark.parametrize("shape", FWD)
@pytest.mark.parametrize("kind", ["fwd", "dgrad"])
def test_conv_fwd_kernels_fenced_and_deterministic(shape, kind):
    ci, co, D, H, W = shape
    cin, cout = (ci, co) if kind == "fwd" else (co, ci)
    g = torch.Generator(device="cuda").manual_seed(sum(shape))
    x, xb = _fenced(1, cin, D, H, W, -7.0)
    x.storage.copy_(torch.randn(x.storage.numel(), generator=g, device="cuda").to(torch.bfloat16))
    y, yb = _fenced(1, cout, D, H, W, 3.0)
    m, mb = _fenced(1, cout, D, H, W, 5.0)
    m.storage.copy_(torch.randn(m.storage.numel(), generator=g, device="cuda").to(torch.bfloat16))
    w = torch.randn(27 * ci * co, generator=g, device="cuda") * 0.05
    b = torch.randn(max(ci, co), generator=g, device="cuda")
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", cin, cout) // 2, dtype=torch.bfloat16, device="cuda")
    st = _lib.stream_ptr()
    _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, int(kind == "dgrad"), st)
    flags = (_lib.VM_CONV_MASK | _lib.VM_CONV_NOBIAS) if kind == "dgrad" else _lib.VM_CONV_RELU
    outs = []
    for _ in range(3):
        y.storage.zero_()
        _lib.call("vm_conv3d_fwd_tc", x.p(), x.bstride, _lib.ptr(wp), _lib.ptr(b), y.p(), y.bstride,
                  m.p() if kind == "dgrad" else None, m.bstride if kind == "dgrad" else 0, 1, cin, cout, D, H, W,
                  flags, st)
        torch.cuda.synchronize()
        outs.append(y.storage.clone())
    for o in outs[1:]:
        assert torch.equal(outs[0], o)
    for s, big, fill in ((x, xb, -7.0), (y, yb, 3.0), (m, mb, 5.0)):
        assert _canaries_ok(big, s.storage.numel(), fill)
    assert bool((_shell(y) == 0).all())  # the conv writes interiors only


WG = [(16, 16, 5, 6, 40), (48, 16, 4, 6, 64), (32, 32, 3, 4, 64), (64, 64, 4, 6, 34), (96, 32, 2, 2, 256),
      (16, 16, 4, 4, 8), (32, 256, 3, 4, 6)]


@pytest.mark.parametrize("shape", WG)
def test_wgrad_kernels_fenced_and_deterministic(shape):
    ci, co, D, H, W = shape
    g = torch.Generator(device="cuda").manual_seed(100 + sum(shape))
    x, xb = _fenced(1, ci, D, H, W, -7.0)
    gy, gb_ = _fenced(1, co, D, H, W, 3.0)
    for s in (x, gy):
        v = s.storage[: s.bstride].view(s.CG, D + 2, H + 2, W + 2, 8)
        v[:, 1:-1, 1:-1, 1:-1] = torch.randn(v[:, 1:-1, 1:-1, 1:-1].shape, generator=g, device="cuda").to(torch.bfloat16)
    nb = _lib.call_size("vm_conv3d_wgrad_tc_ws", 1, ci, co, D, H, W)
    ws = torch.full((nb // 4 + 64 + 2 * GUARD,), 9.0, device="cuda")
    outs = []
    for _ in range(3):
        gw = torch.zeros(27 * ci * co + 2 * GUARD, device="cuda")
        gb = torch.zeros(co + 2 * GUARD, device="cuda")
        gw[:GUARD] = 1.5
        gw[-GUARD:] = 1.5
        gb[:GUARD] = 2.5
        gb[-GUARD:] = 2.5
        _lib.call("vm_conv3d_wgrad_tc", x.p(), x.bstride, gy.p(), gy.bstride, _lib.ptr(gw[GUARD:]),
                  _lib.ptr(gb[GUARD:]), _lib.ptr(ws[GUARD:]), 1, ci, co, D, H, W, _lib.stream_ptr())
        torch.cuda.synchronize()
        assert bool((gw[:GUARD] == 1.5).all() and (gw[-GUARD:] == 1.5).all())
        assert bool((gb[:GUARD] == 2.5).all() and (gb[-GUARD:] == 2.5).all())
        assert bool((ws[:GUARD] == 9.0).all() and (ws[-GUARD:] == 9.0).all())
        outs.append((gw.clone(), gb.clone()))
    for a, b in outs[1:]:
        assert torch.equal(outs[0][0], a) and torch.equal(outs[0][1], b)
    assert _canaries_ok(xb, x.storage.numel(), -7.0) and _canaries_ok(gb_, gy.storage.numel(), 3.0)
