"""Distributed operators over ShardedTensors (the reference's ops API, ops.py:221-333),
on the GPU kernels of libvoxmesh_sm100.

A reference user's per-op code keeps working: ``conv3d_forward(x, params)`` returns
``(y, tape)``, ``conv3d_backward(gy, tape)`` returns ``(gx, gk, gb)`` with the parameter
gradients all-reduced over the mesh, and pooling / upsampling / concat / relu / softmax are
shard-local.  Blocks are device tensors ``[b, x, y, z, c]``; each op converts them to
channel-blocked padded slabs for the kernels and back.

* f32 specs run the CUDA-core fp32 kernels (``vm_conv3d_fwd_simt`` / ``_wgrad_simt``);
  bf16 specs run the tcgen05 kernels (``vm_conv3d_fwd_tc`` / ``_wgrad_tc``) with fp32
  accumulation; f64 has no GPU path and is rejected.
* The input gradient is computed as the forward conv of the halo-exchanged output gradient
  with flipped, transposed taps (`ops.py:100-114` is its adjoint form: the same sum, in
  another order), so ``conv3d_backward`` exchanges the gradient forward instead of running
  ``exchange_backward_local`` on a padded gradient.
* ``softmax_channels`` / ``concat_channels`` run the row kernels of csrc/dense.cu; the train
  step itself fuses softmax into the head kernel and makes the concat zero-copy.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import halo as _halo
from .errors import HaloError, VoxmeshError
from .sharding import ShardedTensor, TensorSpec

SPATIAL_DIMS = ("x", "y", "z")


@dataclass(frozen=True)
class ConvParams:
    """Odd kxkxk kernel [k,k,k,c_in,c_out] plus bias [c_out]; stride 1, SAME (ops.py:33-60)."""

    kernel: np.ndarray
    bias: np.ndarray

    def __post_init__(self):
        k = self.kernel.shape
        if len(k) != 5 or not (k[0] == k[1] == k[2]):
            raise VoxmeshError(f"kernel must be [k,k,k,c_in,c_out], got {k}")
        if k[0] % 2 == 0:
            raise HaloError(f"even kernel extent {k[0]} is unsupported")
        if self.bias.shape != (k[4],):
            raise VoxmeshError(f"bias shape {self.bias.shape} != ({k[4]},)")
        if not (np.isfinite(self.kernel).all() and np.isfinite(self.bias).all()):
            raise VoxmeshError("non-finite values in conv parameters")

    @property
    def k(self):
        return self.kernel.shape[0]

    @property
    def c_in(self):
        return self.kernel.shape[3]

    @property
    def c_out(self):
        return self.kernel.shape[4]


class ConvTape:
    """Forward context a conv backward needs; consumable exactly once (ops.py:221-237)."""

    def __init__(self, x_st, padded_slabs, params, halo_spec):
        self.x_spec = x_st.spec
        self.layout = x_st.layout
        self.mesh = x_st.mesh
        self.padded_slabs = padded_slabs
        self.params = params
        self.halo_spec = halo_spec
        self._used = False

    def take(self):
        if self._used:
            raise VoxmeshError("conv tape already consumed by a backward pass")
        self._used = True
        return self.padded_slabs


def _out_spec(x_st, c_out=None, spatial_scale=1):
    dims = []
    for n, e in x_st.spec.dims:
        if n in SPATIAL_DIMS:
            e = int(e * spatial_scale)
        if n == "c" and c_out is not None:
            e = c_out
        dims.append((n, e))
    return TensorSpec(tuple(dims), x_st.spec.dtype)


# ------------------------------------------------------------------------- block <-> slab
def _vm_code(dtype):
    import torch

    if dtype == torch.float32:
        return _lib.VM_F32
    if dtype == torch.bfloat16:
        return _lib.VM_BF16
    raise VoxmeshError(f"the GPU ops support f32 and bf16 blocks, not {dtype}")


def _vm_dtype(t):
    return _vm_code(t.dtype)


def _slab(B, C, D, H, W, like):
    from .step import Slab

    return Slab(B, C, D, H, W, like.dtype, like.device)


def _to_slab(dense, padded=False):
    """Dense block [B, D, H, W, C] -> slab; ``padded``: the block already holds the margins."""
    B, D, H, W, C = dense.shape
    m = 0 if padded else 1
    s = _slab(B, C, D - 2 * (1 - m), H - 2 * (1 - m), W - 2 * (1 - m), dense)
    src = dense.float().contiguous()  # the converter reads f32 (bf16 -> f32 -> bf16 is exact)
    _lib.call("vm_dense_to_slab", _lib.ptr(src), _lib.VM_F32, s.p(), _vm_dtype(dense), s.bstride,
              B, C, D, H, W, m, _lib.stream_ptr())
    return s


def _to_dense(s):
    import torch

    out = torch.empty((s.B, s.D, s.H, s.W, s.C), dtype=torch.float32, device=s.storage.device)
    _lib.call("vm_slab_to_dense", s.p(), _vm_code(s.dtype), s.bstride, _lib.ptr(out), _lib.VM_F32, s.B, s.C, s.D,
              s.H, s.W, 1, _lib.stream_ptr())
    return out if s.dtype == torch.float32 else out.to(s.dtype)


def _run_blocks(st, fn, *extra):
    return st.mesh.run(fn, per_worker=(st.blocks,) + extra)


# ------------------------------------------------------------------------- conv
def _device_params(params, like, flip):
    import torch

    w = torch.from_numpy(np.ascontiguousarray(params.kernel, dtype=np.float32)).to(like.device)
    b = torch.from_numpy(np.ascontiguousarray(params.bias, dtype=np.float32)).to(like.device)
    ci, co = params.c_in, params.c_out
    if like.dtype == torch.bfloat16:
        cin, cout = (co, ci) if flip else (ci, co)
        wp = torch.empty(_lib.call_size("vm_packed_weights_bytes", cin, cout) // 2, dtype=torch.bfloat16,
                         device=like.device)
        _lib.call("vm_pack_weights", _lib.ptr(w), _lib.ptr(wp), ci, co, int(flip), _lib.stream_ptr())
        return wp, b, w
    if flip:
        wt = torch.empty_like(w)
        _lib.call("vm_weight_flip_transpose", _lib.ptr(w), _lib.ptr(wt), params.k, ci, co, _lib.stream_ptr())
        return wt, b, w
    return w, b, w


def _conv_slab(xs, params, ys, flags, flip=False, mask=None):
    """ys <- conv(xs) on slabs (xs margins already filled)."""
    import torch

    wop, b, _ = _device_params(params, xs.storage, flip)
    cin, cout = (params.c_out, params.c_in) if flip else (params.c_in, params.c_out)
    if xs.dtype == torch.bfloat16:
        _lib.call("vm_conv3d_fwd_tc", xs.p(), xs.bstride, _lib.ptr(wop), _lib.ptr(b), ys.p(), ys.bstride,
                  mask.p() if mask is not None else None, mask.bstride if mask is not None else 0, xs.B, cin, cout,
                  xs.D, xs.H, xs.W, flags, _lib.stream_ptr())
    else:
        _lib.call("vm_conv3d_fwd_simt", _lib.VM_F32, xs.p(), xs.bstride, _lib.ptr(wop), _lib.ptr(b), ys.p(),
                  ys.bstride, mask.p() if mask is not None else None, mask.bstride if mask is not None else 0, xs.B,
                  cin, cout, xs.D, xs.H, xs.W, flags, _lib.stream_ptr())


def conv3d_forward(x: ShardedTensor, params: ConvParams, phase_barrier=True):
    """SAME-padded stride-1 distributed conv (ops.py:251-264); returns (output, tape)."""
    if params.k != 3:
        raise VoxmeshError(f"the GPU conv supports k = 3, got {params.k}")
    spec = _halo.HaloSpec.for_kernel(params.k)
    dims = _halo.dim_axes(x.spec, x.layout)

    def fn(ctx, block):
        padded = _halo.exchange_local(ctx, dims, spec, _halo._FWD_TAG, phase_barrier, block)
        xs = _to_slab(padded.data, padded=True)
        ys = _slab(xs.B, params.c_out, xs.D, xs.H, xs.W, block)
        _conv_slab(xs, params, ys, 0)
        return xs, _to_dense(ys)

    res = _run_blocks(x, fn)
    out = ShardedTensor(_out_spec(x, c_out=params.c_out), x.layout, x.mesh, [None if r is None else r[1] for r in res])
    return out, ConvTape(x, [None if r is None else r[0] for r in res], params, spec)


def conv3d_backward(gout: ShardedTensor, tape: ConvTape, phase_barrier=True):
    """Returns (grad_x, grad_kernel, grad_bias); parameter gradients all-reduced over the
    mesh (ops.py:267-285)."""
    import torch

    slabs = tape.take()
    params = tape.params
    dims = _halo.dim_axes(gout.spec, gout.layout)

    def fn(ctx, gblock, xs):
        # weight gradient first: it needs the gradient slab with zero margins
        gs = _to_slab(gblock)
        ci, co = params.c_in, params.c_out
        gw = torch.zeros(27 * ci * co, dtype=torch.float32, device=gblock.device)
        gb = torch.zeros(co, dtype=torch.float32, device=gblock.device)
        if gblock.dtype == torch.bfloat16:
            nb = _lib.call_size("vm_conv3d_wgrad_tc_ws", xs.B, ci, co, xs.D, xs.H, xs.W)
            ws = torch.empty(nb // 4 + 64, dtype=torch.float32, device=gblock.device)
            _lib.call("vm_conv3d_wgrad_tc", xs.p(), xs.bstride, gs.p(), gs.bstride, _lib.ptr(gw), _lib.ptr(gb),
                      _lib.ptr(ws), xs.B, ci, co, xs.D, xs.H, xs.W, _lib.stream_ptr())
        else:
            nb = _lib.call_size("vm_conv3d_wgrad_simt_ws", xs.B, ci, co, xs.D, xs.H, xs.W)
            ws = torch.empty(nb // 4 + 64, dtype=torch.float32, device=gblock.device)
            _lib.call("vm_conv3d_wgrad_simt", _lib.VM_F32, xs.p(), xs.bstride, gs.p(), gs.bstride, _lib.ptr(gw),
                      _lib.ptr(gb), _lib.ptr(ws), xs.B, ci, co, xs.D, xs.H, xs.W, _lib.stream_ptr())
        # input gradient: forward conv of the halo'd output gradient with flipped taps
        padded = _halo.exchange_local(ctx, dims, tape.halo_spec, _halo._BWD_TAG, phase_barrier, gblock)
        gps = _to_slab(padded.data, padded=True)
        gxs = _slab(xs.B, ci, xs.D, xs.H, xs.W, gblock)
        _conv_slab(gps, params, gxs, _lib.VM_CONV_NOBIAS, flip=True)
        gk = ctx.all_reduce_sum(gw, tag="gk").reshape(params.kernel.shape)
        gbb = ctx.all_reduce_sum(gb, tag="gb")
        return _to_dense(gxs), gk.cpu().numpy(), gbb.cpu().numpy()

    res = gout.mesh.run(fn, per_worker=(gout.blocks, slabs))
    gx = ShardedTensor(tape.x_spec, tape.layout, tape.mesh, [None if r is None else r[0] for r in res])
    first = next(r for r in res if r is not None)
    return gx, first[1].astype(params.kernel.dtype), first[2].astype(params.bias.dtype)


# ------------------------------------------------------------------------- shard-local ops
def maxpool2_forward(x: ShardedTensor):
    """2^3 max pool, first-in-scan-order ties (ops.py:141-156, :288-291); the tape keeps
    the input blocks (the argmax is recomputed in the backward kernel)."""

    def fn(ctx, b):
        xs = _to_slab(b)
        ys = _slab(xs.B, xs.C, xs.D // 2, xs.H // 2, xs.W // 2, b)
        _lib.call("vm_maxpool2_fwd", _vm_dtype(b), xs.p(), xs.bstride, ys.p(), ys.bstride, xs.B, xs.C, xs.D, xs.H,
                  xs.W, _lib.stream_ptr())
        return _to_dense(ys)

    res = _run_blocks(x, fn)
    out = ShardedTensor(_out_spec(x, spatial_scale=0.5), x.layout, x.mesh, res)
    return out, (list(x.blocks), x.spec)


def maxpool2_backward(gout: ShardedTensor, tape):
    """Route each gradient to its cell's argmax (ops.py:159-168, :294-300)."""
    x_blocks, in_spec = tape

    def fn(ctx, g, xb):
        xs, gs = _to_slab(xb), _to_slab(g)
        out = _slab(xs.B, xs.C, xs.D, xs.H, xs.W, xb)
        _lib.call("vm_maxpool2_bwd", _vm_dtype(xb), xs.p(), xs.bstride, gs.p(), gs.bstride, None, 0, out.p(),
                  out.bstride, xs.B, xs.C, xs.D, xs.H, xs.W, 0, _lib.stream_ptr())
        return _to_dense(out)

    res = gout.mesh.run(fn, per_worker=(gout.blocks, x_blocks))
    return ShardedTensor(in_spec, gout.layout, gout.mesh, res)


def upsample2_forward(x: ShardedTensor):
    """Nearest x2 (ops.py:171-173, :303-305)."""

    def fn(ctx, b):
        xs = _to_slab(b)
        ys = _slab(xs.B, xs.C, 2 * xs.D, 2 * xs.H, 2 * xs.W, b)
        _lib.call("vm_upsample2_fwd", _vm_dtype(b), xs.p(), xs.bstride, ys.p(), ys.bstride, xs.B, xs.C, xs.D, xs.H,
                  xs.W, _lib.stream_ptr())
        return _to_dense(ys)

    return ShardedTensor(_out_spec(x, spatial_scale=2), x.layout, x.mesh, _run_blocks(x, fn))


def upsample2_backward(gout: ShardedTensor):
    """Sum of each 2^3 cell (ops.py:176-179, :308-310)."""

    def fn(ctx, g):
        gs = _to_slab(g)
        out = _slab(gs.B, gs.C, gs.D // 2, gs.H // 2, gs.W // 2, g)
        _lib.call("vm_upsample2_bwd", _vm_dtype(g), gs.p(), gs.bstride, None, 0, out.p(), out.bstride, gs.B, gs.C,
                  out.D, out.H, out.W, _lib.stream_ptr())
        return _to_dense(out)

    return ShardedTensor(_out_spec(gout, spatial_scale=0.5), gout.layout, gout.mesh, _run_blocks(gout, fn))


def concat_channels(a: ShardedTensor, b: ShardedTensor):
    """[a, b] along channels (unet.py:215, ops.py:313-323) through ``vm_concat_rows``."""
    import torch

    if a.spec.shape[:-1] != b.spec.shape[:-1] or a.layout.assignments != b.layout.assignments:
        raise VoxmeshError(f"concat needs matching spatial shape and layout: {a.spec.shape} vs {b.spec.shape}")
    if a.spec.dtype != b.spec.dtype:
        raise VoxmeshError(f"concat needs one dtype, got {a.spec.dtype} and {b.spec.dtype}")

    def fn(ctx, x, y):
        x, y = x.contiguous(), y.contiguous()
        out = torch.empty(tuple(x.shape[:-1]) + (x.shape[-1] + y.shape[-1],), dtype=x.dtype, device=x.device)
        rows = x.numel() // x.shape[-1]
        _lib.call("vm_concat_rows", _lib.ptr(x), x.shape[-1] * x.element_size(), _lib.ptr(y),
                  y.shape[-1] * y.element_size(), _lib.ptr(out), rows, _lib.stream_ptr())
        return out

    res = a.mesh.run(fn, per_worker=(a.blocks, b.blocks))
    c_out = a.spec.extent("c") + b.spec.extent("c")
    return ShardedTensor(_out_spec(a, c_out=c_out), a.layout, a.mesh, res)


def relu(x: ShardedTensor):
    """max(x, 0) = x * (x > 0) (ops.py:182-183) through ``vm_relu_mask``."""

    def fn(ctx, b):
        xs = _to_slab(b)
        out = _slab(xs.B, xs.C, xs.D, xs.H, xs.W, b)
        _lib.call("vm_relu_mask", _vm_dtype(b), xs.p(), xs.bstride, xs.p(), xs.bstride, out.p(), out.bstride, xs.B,
                  xs.C, xs.D, xs.H, xs.W, _lib.stream_ptr())
        return _to_dense(out)

    return ShardedTensor(x.spec, x.layout, x.mesh, _run_blocks(x, fn))


def relu_backward(gout: ShardedTensor, x: ShardedTensor):
    """g * (x > 0) (ops.py:186-187) through ``vm_relu_mask``."""

    def fn(ctx, g, xb):
        gs, xs = _to_slab(g), _to_slab(xb)
        out = _slab(gs.B, gs.C, gs.D, gs.H, gs.W, g)
        _lib.call("vm_relu_mask", _vm_dtype(g), gs.p(), gs.bstride, xs.p(), xs.bstride, out.p(), out.bstride, gs.B,
                  gs.C, gs.D, gs.H, gs.W, _lib.stream_ptr())
        return _to_dense(out)

    return ShardedTensor(gout.spec, gout.layout, gout.mesh, gout.mesh.run(fn, per_worker=(gout.blocks, x.blocks)))


def softmax_channels(x: ShardedTensor):
    """Stable channel softmax (ops.py:190-194, :331-333) through ``vm_softmax_rows``."""
    import torch

    def fn(ctx, b):
        b = b.contiguous()
        out = torch.empty_like(b)
        _lib.call("vm_softmax_rows", _vm_dtype(b), _lib.ptr(b), _lib.ptr(out), b.numel() // b.shape[-1], b.shape[-1],
                  _lib.stream_ptr())
        return out

    return ShardedTensor(x.spec, x.layout, x.mesh, _run_blocks(x, fn))
