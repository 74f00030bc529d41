"""tcgen05 conv3d (forward / dgrad operand) vs the CUDA-core kernel and the f64 oracle."""

import numpy as np
import pytest
import torch

from oracle import voxmesh_oracle as O
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.step import Slab
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu

SHAPES = [
    # B, Cin, Cout, D, H, W
    (1, 16, 16, 16, 16, 16),
    (1, 1, 16, 16, 16, 16),
    (1, 48, 16, 12, 16, 16),
    (2, 32, 64, 8, 12, 16),
    (1, 64, 128, 8, 8, 8),
    (1, 128, 64, 8, 8, 8),
    (1, 16, 48, 16, 20, 24),
    (1, 24, 8, 6, 6, 6),
    (1, 16, 16, 32, 32, 128),
    # kd-stacked sweep kernel (Cout <= 48): single planes, segments, ring wrap-around,
    # several units per CTA, odd channel counts
    (1, 8, 16, 1, 9, 9),
    (1, 16, 24, 2, 5, 7),
    (2, 16, 16, 40, 8, 8),
    (1, 32, 32, 40, 24, 24),
    (1, 16, 3, 5, 6, 7),
    (3, 16, 16, 3, 30, 30),
    (1, 8, 48, 70, 4, 4),
    # wide layers of the cfg3/cfg4 ladders: several 256-column N chunks, Cout > 1024 (the dgrad
    # of a 1536-channel concat input), Cin 512
    (1, 16, 1040, 2, 4, 4),
    (1, 512, 256, 2, 4, 6),
]


def _slab_from(x):
    B, D, H, W, C = x.shape
    s = Slab(B, C, D, H, W, torch.bfloat16, "cuda")
    xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    _lib.call("vm_dense_to_slab", _lib.ptr(xt), _lib.VM_F32, s.p(), _lib.VM_BF16, s.bstride, B, C, D, H, W, 1,
              _lib.stream_ptr())
    return s


def _conv_tc(xs, w, b, cout, flags=_lib.VM_CONV_RELU, mask=None, flip=False):
    B, D, H, W = xs.B, xs.D, xs.H, xs.W
    cin_layer, cout_layer = w.shape[3], w.shape[4]
    cin = xs.C
    wt = torch.from_numpy(np.ascontiguousarray(w, np.float32)).cuda()
    nbytes = _lib.call_size("vm_packed_weights_bytes", cin, cout)
    wp = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda")
    _lib.call("vm_pack_weights", _lib.ptr(wt), _lib.ptr(wp), cin_layer, cout_layer, int(flip), _lib.stream_ptr())
    ys = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
    bt = torch.from_numpy(np.ascontiguousarray(b, np.float32)).cuda()
    _lib.call("vm_conv3d_fwd_tc", xs.p(), xs.bstride, _lib.ptr(wp), _lib.ptr(bt), ys.p(), ys.bstride,
              mask.p() if mask is not None else None, mask.bstride if mask is not None else 0,
              B, cin, cout, D, H, W, flags, _lib.stream_ptr())
    return ys


def _conv_simt(xs, w, b, cout, flags=_lib.VM_CONV_RELU, mask=None):
    B, D, H, W = xs.B, xs.D, xs.H, xs.W
    wt = torch.from_numpy(np.ascontiguousarray(w, np.float32)).cuda()
    bt = torch.from_numpy(np.ascontiguousarray(b, np.float32)).cuda()
    ys = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
    _lib.call("vm_conv3d_fwd_simt", _lib.VM_BF16, xs.p(), xs.bstride, _lib.ptr(wt), _lib.ptr(bt), ys.p(), ys.bstride,
              mask.p() if mask is not None else None, mask.bstride if mask is not None else 0,
              B, xs.C, cout, D, H, W, flags, _lib.stream_ptr())
    return ys


@pytest.mark.parametrize("shape", SHAPES)
def test_tc_forward_matches_simt_and_oracle(shape):
    B, cin, cout, D, H, W = shape
    rng = np.random.default_rng(sum(shape))
    x = O.bf16_round(rng.standard_normal((B, D, H, W, cin)).astype(np.float32))
    w = O.bf16_round(rng.uniform(-1, 1, (3, 3, 3, cin, cout)).astype(np.float32) / np.sqrt(27 * cin))
    b = rng.standard_normal(cout).astype(np.float32) * 0.1
    xs = _slab_from(x)
    got = _conv_tc(xs, w, b, cout).interior().cpu().numpy()
    ref = _conv_simt(xs, w, b, cout).interior().cpu().numpy()
    assert rel_l2(got, ref) <= 2e-3
    dense = np.maximum(O.conv3d_dense(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64)), 0)
    assert rel_l2(got, dense) <= 1e-2


def test_tc_forward_keeps_margins_zero():
    B, cin, cout, D, H, W = 1, 16, 16, 10, 12, 14
    rng = np.random.default_rng(3)
    x = rng.standard_normal((B, D, H, W, cin)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (3, 3, 3, cin, cout)).astype(np.float32)
    ys = _conv_tc(_slab_from(x), w, np.ones(cout, np.float32), cout, flags=0)
    torch.cuda.synchronize()
    full = ys.storage[: B * 2 * ys.plane].float().reshape(B, 2, D + 2, H + 2, W + 2, 8).cpu().numpy()
    inner = np.zeros_like(full, dtype=bool)
    inner[:, :, 1:-1, 1:-1, 1:-1] = True
    assert not full[~inner].any()


def test_tc_dgrad_operand_with_relu_mask_matches_oracle_adjoint():
    # dgrad of conv(x; W) for output gradient g = conv(g_pad; flip(W)^T), masked by y>0
    B, cin, cout, D, H, W = 1, 32, 16, 8, 10, 12
    rng = np.random.default_rng(11)
    g = O.bf16_round(rng.standard_normal((B, D, H, W, cout)).astype(np.float32))
    w = O.bf16_round(rng.uniform(-1, 1, (3, 3, 3, cin, cout)).astype(np.float32) / 20)
    m = O.bf16_round(rng.standard_normal((B, D, H, W, cin)).astype(np.float32))
    gs, ms = _slab_from(g), _slab_from(m)
    got = _conv_tc(gs, w, np.zeros(cin, np.float32), cin, flags=_lib.VM_CONV_MASK | _lib.VM_CONV_NOBIAS,
                   mask=ms, flip=True).interior().cpu().numpy()
    xdummy = np.zeros((B, D, H, W, cin))
    gx, _, _ = O.conv3d_dense_backward(g.astype(np.float64), xdummy, w.astype(np.float64))
    ref = np.where(m > 0, gx, 0.0)
    assert rel_l2(got, ref) <= 1e-2


WG_SHAPES = [
    (1, 16, 16, 16, 16, 16),
    (1, 1, 16, 16, 16, 16),
    (1, 48, 16, 12, 16, 16),
    (2, 32, 64, 8, 12, 16),
    (1, 64, 128, 8, 8, 8),
    (1, 128, 64, 8, 8, 8),
    (1, 16, 48, 16, 20, 24),
    (1, 24, 8, 6, 6, 6),
    # wide rows (W >= 32): the "runs" staging mode
    (1, 16, 16, 4, 8, 128),
    (1, 48, 16, 4, 6, 64),
    (1, 32, 32, 6, 8, 64),
    (2, 16, 32, 4, 4, 40),
    (1, 1, 16, 4, 6, 126),
    # kd-along-N kernel (Cout <= 48, W >= 32): padded co groups, several M-tile groups,
    # deep volumes (kd slices reaching outside the sample)
    (1, 16, 48, 5, 6, 40),
    (2, 24, 8, 3, 5, 34),
    (1, 96, 32, 4, 4, 64),
    (1, 8, 16, 40, 4, 32),
    # 256-wide rows: K chunks of 256 anchors (NKK = 16), and the decoder's 96 -> 32 shape whose
    # gy slices only double-buffer at shorter K chunks
    (1, 32, 32, 3, 2, 256),
    (1, 96, 32, 2, 2, 256),
    # Cout 64..80: one kw tap per CTA (three accumulators of N = 3*Nc exceed TMEM)
    (1, 64, 64, 6, 6, 34),
    (1, 32, 64, 4, 8, 40),
    (2, 16, 80, 3, 4, 48),
    # Cout > 160: output-channel chunks of 128 (3 kw x Nc TMEM columns per M-tile), a ragged
    # last chunk, no ones slot (separate bias partials)
    (1, 32, 256, 4, 6, 8),
    (1, 64, 200, 3, 4, 6),
    (1, 128, 512, 2, 4, 4),
    # whole 128-channel chunks run as CTA columns of one launch: a ones slot (9*CG % 16 != 0),
    # two samples, and the depth-split block of cfg3's deepest level (one wave, no K split)
    (2, 72, 384, 3, 4, 10),
    (1, 512, 512, 2, 16, 16),
]


def _wgrad(fn, xs, gs, cin, cout):
    B, D, H, W = xs.B, xs.D, xs.H, xs.W
    gw = torch.zeros(27 * cin * cout, dtype=torch.float32, device="cuda")
    gb = torch.zeros(cout, dtype=torch.float32, device="cuda")
    if fn == "vm_conv3d_wgrad_tc":
        nb = _lib.call_size("vm_conv3d_wgrad_tc_ws", B, cin, cout, D, H, W)
        ws = torch.empty(nb // 4 + 64, dtype=torch.float32, device="cuda")
        _lib.call(fn, xs.p(), xs.bstride, gs.p(), gs.bstride, _lib.ptr(gw), _lib.ptr(gb), _lib.ptr(ws),
                  B, cin, cout, D, H, W, _lib.stream_ptr())
    else:
        nb = _lib.call_size("vm_conv3d_wgrad_simt_ws", B, cin, cout, D, H, W)
        ws = torch.empty(nb // 4 + 64, dtype=torch.float32, device="cuda")
        _lib.call(fn, _lib.VM_BF16, xs.p(), xs.bstride, gs.p(), gs.bstride, _lib.ptr(gw), _lib.ptr(gb),
                  _lib.ptr(ws), B, cin, cout, D, H, W, _lib.stream_ptr())
    torch.cuda.synchronize()
    return gw.cpu().numpy().reshape(3, 3, 3, cin, cout), gb.cpu().numpy()


@pytest.mark.parametrize("shape", WG_SHAPES)
def test_tc_wgrad_matches_simt_and_oracle(shape):
    B, cin, cout, D, H, W = shape
    rng = np.random.default_rng(100 + sum(shape))
    x = O.bf16_round(rng.standard_normal((B, D, H, W, cin)).astype(np.float32))
    g = O.bf16_round(rng.standard_normal((B, D, H, W, cout)).astype(np.float32))
    xs, gs = _slab_from(x), _slab_from(g)
    gw, gb = _wgrad("vm_conv3d_wgrad_tc", xs, gs, cin, cout)
    sw, sb = _wgrad("vm_conv3d_wgrad_simt", xs, gs, cin, cout)
    assert rel_l2(gw, sw) <= 1e-5 and rel_l2(gb, sb) <= 1e-5
    _, rgk, rgb = O.conv3d_dense_backward(g.astype(np.float64), x.astype(np.float64),
                                           np.zeros((3, 3, 3, cin, cout)))
    assert rel_l2(gw, rgk) <= 1e-5
    assert rel_l2(gb, rgb) <= 1e-5


def test_batched_repack_equals_single_packs():
    # vm_pack_weights_batch (one launch, every layer, both operands) == vm_pack_weights per job
    shapes = [(1, 16), (16, 16), (48, 16), (16, 32), (96, 32), (64, 128), (128, 64), (24, 8), (16, 48)]
    rng = np.random.default_rng(5)
    ws, bufs, refs, rows, begin = [], [], [], [], 0
    for cin, cout in shapes:
        w = torch.from_numpy(rng.standard_normal(27 * cin * cout).astype(np.float32)).cuda()
        ws.append(w)
        for flip in (0, 1):
            ci, co = (cout, cin) if flip else (cin, cout)
            n = _lib.call_size("vm_packed_weights_bytes", ci, co) // 2
            ref = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(ref), cin, cout, flip, _lib.stream_ptr())
            buf = torch.full((n,), float("nan"), dtype=torch.bfloat16, device="cuda")
            refs.append(ref)
            bufs.append(buf)
            rows.append((w.data_ptr(), buf.data_ptr(), cin, cout, flip, 0, begin))
            begin += n
    dt = np.dtype([("w", "<u8"), ("packed", "<u8"), ("cin", "<i4"), ("cout", "<i4"), ("flip", "<i4"),
                   ("pad", "<i4"), ("begin", "<i8")])
    jobs = torch.from_numpy(np.array(rows, dtype=dt).view(np.uint8).copy()).cuda()
    _lib.call("vm_pack_weights_batch", _lib.ptr(jobs), len(rows), begin, _lib.stream_ptr())
    torch.cuda.synchronize()
    for ref, buf in zip(refs, bufs):
        assert torch.equal(ref.view(torch.int16), buf.view(torch.int16))


def test_dgrad_composite_and_plane_ranges_are_the_kernels():
    # vm_conv3d_dgrad (csrc/abi.cu) == the flipped-operand tc conv with the ReLU mask, and
    # vm_conv3d_fwd_tc_range over [0,1) + [1,D-1) + [D-1,D) (the halo-overlap split) == one
    # full launch, bitwise, for the sweep (thin) and the general kernels
    for (B, cin, cout, D, H, W) in ((1, 16, 32, 10, 8, 40), (2, 64, 128, 9, 6, 12)):
        rng = np.random.default_rng(21 + cin)
        x = O.bf16_round(rng.standard_normal((B, D, H, W, cin)).astype(np.float32))
        g = O.bf16_round(rng.standard_normal((B, D, H, W, cout)).astype(np.float32))
        w = O.bf16_round(rng.uniform(-1, 1, (3, 3, 3, cin, cout)).astype(np.float32) / 20)
        b = rng.standard_normal(cout).astype(np.float32) * 0.1
        xs, gs = _slab_from(x), _slab_from(g)
        ref = _conv_tc(xs, w, b, cout)
        wt = torch.from_numpy(np.ascontiguousarray(w)).cuda()
        wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", cin, cout) // 2, dtype=torch.bfloat16,
                         device="cuda")
        wpt = torch.empty(_lib.call_size("vm_packed_weights_bytes", cout, cin) // 2, dtype=torch.bfloat16,
                          device="cuda")
        _lib.call("vm_pack_weights", _lib.ptr(wt), _lib.ptr(wp), cin, cout, 0, _lib.stream_ptr())
        _lib.call("vm_pack_weights", _lib.ptr(wt), _lib.ptr(wpt), cin, cout, 1, _lib.stream_ptr())
        bt = torch.from_numpy(b).cuda()
        y = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
        for d0, nd in ((1, D - 2), (0, 1), (D - 1, 1)):
            _lib.call("vm_conv3d_fwd_tc_range", xs.p(), xs.bstride, _lib.ptr(wp), _lib.ptr(bt), y.p(), y.bstride,
                      None, 0, B, cin, cout, D, H, W, d0, nd, _lib.VM_CONV_RELU, None, 0, _lib.stream_ptr())
        torch.cuda.synchronize()
        assert torch.equal(y.storage, ref.storage)
        gx = Slab(B, cin, D, H, W, torch.bfloat16, "cuda")
        _lib.call("vm_conv3d_dgrad", gs.p(), gs.bstride, _lib.ptr(wpt), xs.p(), xs.bstride, gx.p(), gx.bstride, B,
                  cin, cout, D, H, W, _lib.stream_ptr())
        gx_ref = _conv_tc(gs, w, np.zeros(cin, np.float32), cin, flags=_lib.VM_CONV_MASK | _lib.VM_CONV_NOBIAS,
                          mask=xs, flip=True)
        torch.cuda.synchronize()
        assert torch.equal(gx.storage, gx_ref.storage)


@pytest.mark.parametrize("shape", [(1, 128, 256, 4, 16, 16), (1, 64, 128, 8, 8, 8), (2, 128, 64, 8, 8, 8),
                                   (1, 256, 512, 4, 4, 4), (1, 512, 512, 2, 16, 16)])
def test_tc_forward_split_k_workspace(shape):
    # vm_conv3d_fwd_tc_ws: shapes with few tile units (<= SMs / 4, the deep levels of a split
    # volume) split the K reduction over CTAs with f32 partials in the caller's scratch; the
    # last split of each tile sums them in split order
    B, cin, cout, D, H, W = shape
    rng = np.random.default_rng(7 + sum(shape))
    x = O.bf16_round(rng.standard_normal((B, D, H, W, cin)).astype(np.float32))
    w = O.bf16_round(rng.uniform(-1, 1, (3, 3, 3, cin, cout)).astype(np.float32) / np.sqrt(27 * cin))
    b = rng.standard_normal(cout).astype(np.float32) * 0.1
    m = O.bf16_round(rng.standard_normal((B, D, H, W, cout)).astype(np.float32))
    xs, ms = _slab_from(x), _slab_from(m)
    wt = torch.from_numpy(np.ascontiguousarray(w, np.float32)).cuda()
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", cin, cout) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.call("vm_pack_weights", _lib.ptr(wt), _lib.ptr(wp), cin, cout, 0, _lib.stream_ptr())
    bt = torch.from_numpy(b).cuda()
    nbytes = _lib.call_size("vm_conv3d_fwd_tc_ws_bytes", B, cin, cout, D, H, W)
    assert nbytes > 0
    ws = torch.zeros(nbytes // 4 + 64, dtype=torch.float32, device="cuda")
    flags = _lib.VM_CONV_RELU | _lib.VM_CONV_MASK
    outs = []
    for use_ws in (False, True, True):
        ys = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
        if use_ws:
            _lib.call("vm_conv3d_fwd_tc_ws", xs.p(), xs.bstride, _lib.ptr(wp), _lib.ptr(bt), ys.p(), ys.bstride,
                      ms.p(), ms.bstride, B, cin, cout, D, H, W, flags, _lib.ptr(ws), nbytes, _lib.stream_ptr())
        else:
            _lib.call("vm_conv3d_fwd_tc", xs.p(), xs.bstride, _lib.ptr(wp), _lib.ptr(bt), ys.p(), ys.bstride,
                      ms.p(), ms.bstride, B, cin, cout, D, H, W, flags, _lib.stream_ptr())
        outs.append(ys.interior().cpu().numpy())
    assert np.array_equal(outs[1], outs[2])          # deterministic
    assert rel_l2(outs[1], outs[0]) <= 5e-3          # same math, other f32 summation order
    dense = np.maximum(O.conv3d_dense(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64)), 0)
    dense = np.where(m > 0, dense, 0)
    assert rel_l2(outs[1], dense) <= 1e-2
    nz = int(torch.count_nonzero(ws[:64]).item())  # tile counters (first 256 B) are back to zero
    assert nz == 0


@pytest.mark.parametrize("shape,split", [((1, 128, 128, 16, 16, 16), 3), ((1, 64, 128, 4, 8, 8), 2),
                                         ((1, 256, 256, 4, 8, 8), 4), ((2, 64, 64, 4, 8, 8), 2)])
def test_tc_forward_cluster_split_k_is_bitwise_the_global_fix_up(shape, split):
    """Opt-in cluster split-K (vm_debug_set_fwd_cluster): the K splits of a tile are one
    thread-block cluster, partials in each CTA's shared memory, the fix-up reads them over DSMEM
    (barrier.cluster + mapa + ld.shared::cluster) — bitwise the global-workspace fix-up (same
    split order), masked epilogue included, and the f64 oracle within the bf16 bound."""
    B, cin, cout, D, H, W = shape
    rng = np.random.default_rng(11 + sum(shape))
    x = O.bf16_round(rng.standard_normal((B, D, H, W, cin)).astype(np.float32))
    w = O.bf16_round(rng.uniform(-1, 1, (3, 3, 3, cin, cout)).astype(np.float32) / np.sqrt(27 * cin))
    b = rng.standard_normal(cout).astype(np.float32) * 0.1
    m = O.bf16_round(rng.standard_normal((B, D, H, W, cout)).astype(np.float32))
    xs, ms = _slab_from(x), _slab_from(m)
    wt = torch.from_numpy(np.ascontiguousarray(w, np.float32)).cuda()
    wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", cin, cout) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.call("vm_pack_weights", _lib.ptr(wt), _lib.ptr(wp), cin, cout, 0, _lib.stream_ptr())
    bt = torch.from_numpy(b).cuda()
    nbytes = _lib.call_size("vm_conv3d_fwd_tc_ws_bytes", B, cin, cout, D, H, W)
    ws = torch.zeros(nbytes // 4 + 64, dtype=torch.float32, device="cuda")
    flags = _lib.VM_CONV_RELU | _lib.VM_CONV_MASK
    lib = _lib.load()
    outs = {}
    try:
        lib.vm_debug_set_fwd_plan(1, 1)
        lib.vm_debug_set_fwd_max_split(16)
        lib.vm_debug_force_fwd_split(split)
        for cl in (1, 0, 1):
            lib.vm_debug_set_fwd_cluster(cl)
            ys = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
            _lib.call("vm_conv3d_fwd_tc_ws", xs.p(), xs.bstride, _lib.ptr(wp), _lib.ptr(bt), ys.p(), ys.bstride,
                      ms.p(), ms.bstride, B, cin, cout, D, H, W, flags, _lib.ptr(ws), nbytes, _lib.stream_ptr())
            torch.cuda.synchronize()
            outs.setdefault(cl, []).append(ys.storage.cpu())
    finally:
        lib.vm_debug_set_fwd_cluster(0)
        lib.vm_debug_force_fwd_split(0)
        lib.vm_debug_set_fwd_plan(0, 0)
    assert torch.equal(outs[1][0], outs[1][1])       # deterministic
    assert torch.equal(outs[1][0], outs[0][0])       # cluster == global fix-up
    ys = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
    ys.storage.copy_(outs[1][0].cuda())
    dense = np.maximum(O.conv3d_dense(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64)), 0)
    dense = np.where(m > 0, dense, 0)
    assert rel_l2(ys.interior().cpu().numpy(), dense) <= 1e-2


C1_SHAPES = [(1, 16, 16, 16, 16), (2, 32, 6, 10, 34), (1, 8, 5, 7, 9), (1, 16, 12, 32, 128), (1, 24, 3, 4, 5)]


@pytest.mark.parametrize("shape", C1_SHAPES)
def test_first_layer_c1_forward_and_wgrad(shape):
    # Cin = 1 im2col kernels (27 taps as K) against the f64 oracle and the channel-blocked path
    B, cout, D, H, W = shape
    rng = np.random.default_rng(21 + sum(shape))
    x = O.bf16_round(rng.standard_normal((B, D, H, W, 1)).astype(np.float32))
    w = O.bf16_round(rng.uniform(-1, 1, (3, 3, 3, 1, cout)).astype(np.float32) / np.sqrt(27))
    b = rng.standard_normal(cout).astype(np.float32) * 0.1
    g = O.bf16_round(rng.standard_normal((B, D, H, W, cout)).astype(np.float32))
    xs, gs = _slab_from(x), _slab_from(g)
    xd = torch.from_numpy(np.ascontiguousarray(x[..., 0], np.float32)).cuda()
    x1 = torch.full((B * (D + 2) * (H + 2) * (W + 2),), float("nan"), dtype=torch.bfloat16, device="cuda")
    _lib.call("vm_dense_to_compact1", _lib.ptr(xd), _lib.ptr(x1), B, D, H, W, _lib.stream_ptr())
    wt = torch.from_numpy(np.ascontiguousarray(w, np.float32)).cuda()
    bt = torch.from_numpy(b).cuda()
    ys = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
    _lib.call("vm_conv3d_fwd_c1", _lib.ptr(x1), 0, _lib.ptr(wt), _lib.ptr(bt), ys.p(), ys.bstride, B, cout, D, H,
              W, _lib.VM_CONV_RELU, _lib.stream_ptr())
    got = ys.interior().cpu().numpy()
    dense = np.maximum(O.conv3d_dense(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64)), 0)
    assert rel_l2(got, dense) <= 1e-2
    if cout % 16 == 0:
        ref = _conv_tc(xs, w, b, cout).interior().cpu().numpy()
        assert rel_l2(got, ref) <= 2e-3
    # margins stay zero (the next conv reads them as padding)
    full = ys.storage[: B * ys.CG * ys.plane].float().reshape(B, ys.CG, D + 2, H + 2, W + 2, 8).cpu().numpy()
    inner = np.zeros_like(full, dtype=bool)
    inner[:, :, 1:-1, 1:-1, 1:-1] = True
    assert not full[~inner].any()
    # weight gradient
    gw = torch.zeros(27 * cout, dtype=torch.float32, device="cuda")
    gb = torch.zeros(cout, dtype=torch.float32, device="cuda")
    nb = _lib.call_size("vm_conv3d_wgrad_c1_ws", B, cout, D, H, W)
    ws = torch.empty(nb // 4 + 64, dtype=torch.float32, device="cuda")
    outs = []
    for _ in range(2):
        _lib.call("vm_conv3d_wgrad_c1", _lib.ptr(x1), 0, gs.p(), gs.bstride, _lib.ptr(gw), _lib.ptr(gb),
                  _lib.ptr(ws), B, cout, D, H, W, _lib.stream_ptr())
        torch.cuda.synchronize()
        outs.append((gw.cpu().numpy().copy(), gb.cpu().numpy().copy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    _, rgk, rgb = O.conv3d_dense_backward(g.astype(np.float64), x.astype(np.float64), np.zeros((3, 3, 3, 1, cout)))
    assert rel_l2(outs[0][0].reshape(3, 3, 3, 1, cout), rgk) <= 1e-5
    assert rel_l2(outs[0][1], rgb) <= 1e-5


def test_wgrad_input_channel_chunks_match_one_call():
    # the multi-group kd weight gradient split into 32-channel chunks (volumes >= 4 M voxels)
    # == the one-call kernel within fp32 summation-order tolerance, bias written once
    B, cin, cout, D, H, W = 1, 96, 32, 64, 256, 256
    g = torch.Generator(device="cuda").manual_seed(5)
    xs = Slab(B, cin, D, H, W, torch.bfloat16, "cuda")
    gs = Slab(B, cout, D, H, W, torch.bfloat16, "cuda")
    for s in (xs, gs):
        v = s.storage[: s.bstride].view(s.CG, D + 2, H + 2, W + 2, 8)
        v[:, 1:-1, 1:-1, 1:-1] = torch.randn(v[:, 1:-1, 1:-1, 1:-1].shape, generator=g, device="cuda").to(torch.bfloat16)
    lib = _lib.load()
    res = []
    for chunk in (0, 1):
        lib.vm_debug_set_wgrad_chunk(chunk)
        try:
            gw = torch.zeros(27 * cin * cout, device="cuda")
            gb = torch.full((cout,), 7.0, device="cuda")
            nb = _lib.call_size("vm_conv3d_wgrad_tc_ws", B, cin, cout, D, H, W)
            ws = torch.empty(nb // 4 + 64, device="cuda")
            _lib.call("vm_conv3d_wgrad_tc", xs.p(), xs.bstride, gs.p(), gs.bstride, _lib.ptr(gw), _lib.ptr(gb),
                      _lib.ptr(ws), B, cin, cout, D, H, W, _lib.stream_ptr())
            torch.cuda.synchronize()
            res.append((gw.double(), gb.double()))
        finally:
            lib.vm_debug_set_wgrad_chunk(1)
    assert float((res[0][0] - res[1][0]).norm() / res[0][0].norm()) <= 1e-3
    assert float((res[0][1] - res[1][1]).norm() / res[0][1].norm()) <= 1e-3
