"""The reference's per-op API on ShardedTensors (ops.py:221-333), GPU kernels vs the f64
oracle, on a 2x2 threads mesh on one GPU (halo exchange included)."""

import numpy as np
import pytest
import torch

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu

AXES = [("mx", 2), ("my", 2)]
LAYOUT = {"x": "mx", "y": "my"}


def _mesh():
    return vm.create_mesh(AXES, backend="threads")


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-5), ("bf16", 1e-2)])
def test_conv3d_forward_backward(dtype, tol):
    rng = np.random.default_rng(7)
    B, D, H, W, ci, co = 1, 8, 8, 12, 16, 24
    x = rng.standard_normal((B, D, H, W, ci)).astype(np.float32)
    k = (rng.uniform(-1, 1, (3, 3, 3, ci, co)) / np.sqrt(27 * ci)).astype(np.float32)
    b = (0.1 * rng.standard_normal(co)).astype(np.float32)
    g = rng.standard_normal((B, D, H, W, co)).astype(np.float32)
    if dtype == "bf16":
        x, k, g = O.bf16_round(x), O.bf16_round(k), O.bf16_round(g)
    with _mesh() as mesh:
        spec = vm.TensorSpec((("batch", B), ("x", D), ("y", H), ("z", W), ("c", ci)), dtype)
        gspec = vm.TensorSpec((("batch", B), ("x", D), ("y", H), ("z", W), ("c", co)), dtype)
        xs = vm.shard(x, spec, vm.Layout(LAYOUT), mesh)
        params = vm.ConvParams(k, b)
        y, tape = vm.conv3d_forward(xs, params)
        gx, gk, gb = vm.conv3d_backward(vm.shard(g, gspec, vm.Layout(LAYOUT), mesh), tape)
        yg = vm.gather(y).astype(np.float64)
        gxg = vm.gather(gx).astype(np.float64)
        with pytest.raises(vm.VoxmeshError):
            vm.conv3d_backward(vm.shard(g, gspec, vm.Layout(LAYOUT), mesh), tape)
    ry = O.conv3d_dense(x.astype(np.float64), k.astype(np.float64), b.astype(np.float64))
    rgx, rgk, rgb = O.conv3d_dense_backward(g.astype(np.float64), x.astype(np.float64), k.astype(np.float64))
    assert rel_l2(yg, ry) <= tol
    assert rel_l2(gxg, rgx) <= tol
    assert rel_l2(gk, rgk) <= tol and rel_l2(gb, rgb) <= tol
    assert gk.shape == k.shape and gb.shape == b.shape


def test_shard_local_ops_match_oracle():
    rng = np.random.default_rng(3)
    B, D, H, W, C = 1, 8, 8, 8, 8
    x = rng.standard_normal((B, D, H, W, C)).astype(np.float32)
    with _mesh() as mesh:
        lay = vm.Layout(LAYOUT)
        spec = vm.TensorSpec((("batch", B), ("x", D), ("y", H), ("z", W), ("c", C)), "f32")
        xs = vm.shard(x, spec, lay, mesh)
        p, ptape = vm.maxpool2_forward(xs)
        pg = rng.standard_normal(p.spec.shape).astype(np.float32)
        gin = vm.maxpool2_backward(vm.shard(pg, p.spec, lay, mesh), ptape)
        up = vm.upsample2_forward(p)
        upb = vm.upsample2_backward(vm.shard(x, spec, lay, mesh))
        r = vm.relu(xs)
        rb = vm.relu_backward(vm.shard(pg.repeat(2, 1).repeat(2, 2).repeat(2, 3), spec, lay, mesh), xs)
        cat = vm.concat_channels(xs, r)
        sm = vm.softmax_channels(xs)
        got = {n: vm.gather(t) for n, t in (("p", p), ("gin", gin), ("up", up), ("upb", upb), ("r", r),
                                              ("rb", rb), ("cat", cat), ("sm", sm))}
    rp, idx = O.maxpool2_dense(x)
    assert np.array_equal(got["p"], rp)
    assert np.array_equal(got["gin"], O.maxpool2_dense_backward(pg, idx, x.shape))
    assert np.array_equal(got["up"], O.upsample2_dense(rp))
    assert rel_l2(got["upb"], O.upsample2_dense_backward(x.astype(np.float64))) <= 1e-6
    assert np.array_equal(got["r"], np.maximum(x, 0))
    gfull = pg.repeat(2, 1).repeat(2, 2).repeat(2, 3)
    assert np.array_equal(got["rb"], np.where(x > 0, gfull, 0))
    assert np.array_equal(got["cat"], np.concatenate([x, np.maximum(x, 0)], axis=-1))
    assert rel_l2(got["sm"], O.softmax_dense(x.astype(np.float64))) <= 1e-6


def test_distributed_losses_match_oracle():
    rng = np.random.default_rng(11)
    B, D, H, W, C = 1, 8, 8, 8, 3
    logits = rng.standard_normal((B, D, H, W, C))
    probs = (np.exp(logits) / np.exp(logits).sum(-1, keepdims=True)).astype(np.float32)
    lab = rng.integers(0, 3, (B, D, H, W))
    oh = vm.one_hot(lab, 3)
    with _mesh() as mesh:
        lay = vm.Layout(LAYOUT)
        spec = vm.TensorSpec((("batch", B), ("x", D), ("y", H), ("z", W), ("c", C)), "f32")
        ps, gs = vm.shard(probs, spec, lay, mesh), vm.shard(oh, spec, lay, mesh)
        dice = vm.soft_dice_loss(ps, gs)
        ce = vm.cross_entropy_loss(ps, gs)
        comb = vm.combined_loss(vm.LossWeights(), ps, gs)
    st = O.loss_stats(probs.astype(np.float64), oh.astype(np.float64))
    rcomb, rdice, rce = O.losses_from_stats(st, 3, D * H * W)
    assert abs(dice - rdice) <= 1e-9 and abs(ce - rce) <= 1e-9 and abs(comb - rcomb) <= 1e-9


@pytest.mark.parametrize("C,D,H,W", [(16, 4, 6, 8), (24, 3, 5, 7), (32, 8, 8, 8)])
def test_bf16_slab_upsample_and_pool_bit_exact(C, D, H, W):
    # the bf16 slab kernels the train step runs (upsample: one thread per input vector writing
    # the 2x2x2 cell; pool: first max in scan order) against numpy on the same bf16 values
    from paper_1909_03108_b200 import _lib
    from paper_1909_03108_b200.step import Slab
    import torch
    rng = np.random.default_rng(C + D)
    B = 2
    x = O.bf16_round(rng.standard_normal((B, D, H, W, C)).astype(np.float32))

    def to_slab(a):
        b_, d_, h_, w_, c_ = a.shape
        s = Slab(b_, c_, d_, h_, w_, torch.bfloat16, "cuda")
        t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
        _lib.call("vm_dense_to_slab", _lib.ptr(t), _lib.VM_F32, s.p(), _lib.VM_BF16, s.bstride, b_, c_, d_, h_, w_, 1,
                  _lib.stream_ptr())
        return s

    xs = to_slab(x)
    ys = Slab(B, C, 2 * D, 2 * H, 2 * W, torch.bfloat16, "cuda")
    _lib.call("vm_upsample2_fwd", _lib.VM_BF16, xs.p(), xs.bstride, ys.p(), ys.bstride, B, C, D, H, W,
              _lib.stream_ptr())
    up = ys.interior().float().cpu().numpy()
    assert np.array_equal(up, x.repeat(2, 1).repeat(2, 2).repeat(2, 3))
    ps = Slab(B, C, D // 2, H // 2, W // 2, torch.bfloat16, "cuda") if D % 2 == 0 and H % 2 == 0 and W % 2 == 0 else None
    if ps is not None:
        _lib.call("vm_maxpool2_fwd", _lib.VM_BF16, xs.p(), xs.bstride, ps.p(), ps.bstride, B, C, D, H, W,
                  _lib.stream_ptr())
        rp, _ = O.maxpool2_dense(x)
        assert np.array_equal(ps.interior().float().cpu().numpy(), rp)


def test_sgd_momentum_bitwise_and_nonfinite_skip():
    # vm_sgd_momentum (training.py:202-219): numpy fp32 op order per element, layers with
    # non-finite gradients skipped entirely; odd layer sizes exercise the 4-wide path's edges
    from paper_1909_03108_b200 import _lib
    rng = np.random.default_rng(17)
    sizes = [5, 4096 + 3, 7, 12, 1025, 64]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(off[-1])
    p = rng.standard_normal(n).astype(np.float32)
    v = rng.standard_normal(n).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    g[off[1] + 100] = np.nan  # layer 1 is skipped
    g[off[4] + 3] = np.inf    # layer 4 is skipped
    lr, mu = np.float32(0.01), np.float32(0.9)
    pt, vt, gt = (torch.from_numpy(a.copy()).cuda() for a in (p, v, g))
    ot = torch.from_numpy(off).cuda()
    flags = torch.zeros(len(sizes), dtype=torch.int32, device="cuda")
    _lib.call("vm_sgd_momentum", _lib.ptr(pt), _lib.ptr(vt), _lib.ptr(gt), _lib.ptr(ot), len(sizes), max(sizes),
              _lib.ptr(flags), float(lr), float(mu), _lib.stream_ptr())
    torch.cuda.synchronize()
    rp, rv = p.copy(), v.copy()
    for li, (a, b) in enumerate(zip(off[:-1], off[1:])):
        if not np.isfinite(g[a:b]).all():
            continue
        rv[a:b] = rv[a:b] * mu
        rv[a:b] = rv[a:b] + g[a:b]
        rp[a:b] = rp[a:b] - lr * rv[a:b]
    assert np.array_equal(pt.cpu().numpy().view(np.uint32), rp.view(np.uint32))
    assert np.array_equal(vt.cpu().numpy().view(np.uint32), rv.view(np.uint32))
    assert flags.cpu().numpy().tolist() == [0, 1, 0, 0, 1, 0]


@pytest.mark.parametrize("nvox,ncls", [(4096, 3), (4095, 3), (1000, 2), (64, 4)])
def test_onehot_u8_kernel(nvox, ncls):
    # vm_onehot_u8 (training.py:68-69 on the GPU): the 4-voxel vector path and the scalar path
    from paper_1909_03108_b200 import _lib
    lab = np.random.default_rng(nvox).integers(0, ncls, nvox).astype(np.uint8)
    lt = torch.from_numpy(lab).cuda()
    oh = torch.full((nvox * ncls,), -1.0, dtype=torch.float32, device="cuda")
    _lib.call("vm_onehot_u8", _lib.ptr(lt), _lib.ptr(oh), nvox, ncls, _lib.stream_ptr())
    assert np.array_equal(oh.cpu().numpy().reshape(nvox, ncls), np.eye(ncls, dtype=np.float32)[lab])
