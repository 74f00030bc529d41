"""Halo exchange of block margins before windowed ops, and its exact adjoint.

Protocol (reference ``voxmesh/halo.py:109-229``), restated on device buffers:
margins are exchanged one spatial dim at a time; the face sent in phase i spans
the margins already filled by phases < i, so edges/corners arrive over 2-3 hops
with no diagonal messages; global-boundary margins are zero; the backward is
the linear adjoint (dims reversed, interior kept, low side added first).

B200 realisation: the padded buffer is allocated once and filled in place
(no ``np.concatenate``, halo.py:148): the interior is written by the producer,
each face is packed into a contiguous message by the ``vm_box_pack`` kernel
(16-byte vectorised), moved by the mesh transport (NCCL send/recv over NVLink in
spmd mode, stream-ordered device queues in threads mode) and written into the
margins by ``vm_box_unpack`` (``vm_box_unpack_add`` for the adjoint).  The same
plan drives the channel-blocked slabs of the U-Net step (:mod:`.step`).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

from . import _lib
from .errors import HaloError
from .sharding import BATCH_DIM, CHANNEL_DIM, ShardedTensor, local_shape, torch_dtype

_FWD_TAG = "halo"
_BWD_TAG = "halo-bwd"


@dataclass(frozen=True)
class HaloSpec:
    """Per-spatial-dim (lo, hi) margins in voxels (halo.py:34-70)."""

    margins: tuple

    def __init__(self, margins):
        if isinstance(margins, dict):
            margins = tuple((d, int(v[0]), int(v[1])) for d, v in sorted(margins.items()))
        else:
            margins = tuple((str(d), int(lo), int(hi)) for d, lo, hi in margins)
        for d, lo, hi in margins:
            if d in (BATCH_DIM, CHANNEL_DIM):
                raise HaloError(f"halo margins only apply to spatial dims, not {d!r}")
            if lo < 0 or hi < 0:
                raise HaloError(f"negative margin on {d!r}: ({lo}, {hi})")
        object.__setattr__(self, "margins", margins)

    @classmethod
    def for_kernel(cls, k, dims=("x", "y", "z")):
        if k % 2 == 0:
            raise HaloError(
                f"even kernel extent {k} is unsupported: margins must be (k-1)/2 per side, which requires odd k"
            )
        m = (k - 1) // 2
        return cls(tuple((d, m, m) for d in dims))

    def margin(self, dim):
        for d, lo, hi in self.margins:
            if d == dim:
                return lo, hi
        return 0, 0

    def total(self, dim):
        lo, hi = self.margin(dim)
        return lo + hi


@dataclass
class PaddedBlock:
    """A block grown by its margins + per-face provenance ("neighbor" | "zero")."""

    data: object
    halo: HaloSpec
    dim_names: tuple
    faces: dict = field(default_factory=dict)

    def interior_slices(self):
        return tuple(
            slice(self.halo.margin(d)[0], self.data.shape[i] - self.halo.margin(d)[1])
            for i, d in enumerate(self.dim_names)
        )

    @property
    def interior(self):
        return self.data[self.interior_slices()]


def dim_axes(spec, layout):
    """((dim, axis or None), ...) in tensor-dim order (halo.py:98-100)."""
    return tuple((n, layout.axis_for(n)) for n in spec.names)


# ---------------------------------------------------------------------------
# Plan: the boxes of every phase, in padded coordinates of a 5-D view
# ---------------------------------------------------------------------------


def _pad5(shape):
    """View any rank-<=5 shape as 5-D (leading ones)."""
    return (1,) * (5 - len(shape)) + tuple(shape)


@dataclass
class Phase:
    axis_pos: int  # index of the phase dim in the 5-D view
    lo: int
    hi: int
    lo_nbr: object
    hi_nbr: object
    send_down: tuple  # (lo5, ext5) of the first `hi` interior rows -> lo neighbour
    send_up: tuple  # last `lo` interior rows -> hi neighbour
    recv_lo: tuple  # margin [0, lo) <- lo neighbour (or zero)
    recv_hi: tuple  # margin [lo+n, lo+n+hi) <- hi neighbour (or zero)


def plan_phases(core5, margins5, nbrs):
    """Phases for a 5-D block of interior shape ``core5`` with per-axis (lo, hi)
    margins ``margins5`` and ``nbrs[axis] = (lo_rank|None, hi_rank|None)``."""
    phases = []
    for i in range(5):
        lo, hi = margins5[i]
        if lo == 0 and hi == 0:
            continue
        n = core5[i]
        if lo > n or hi > n:
            raise HaloError(
                f"margin ({lo},{hi}) exceeds local extent {n}; use a smaller mesh axis or a larger volume"
            )

        def box(a, e):
            lo5, ext5 = [], []
            for j in range(5):
                mlo, mhi = margins5[j]
                if j == i:
                    lo5.append(a)
                    ext5.append(e)
                elif j < i:
                    lo5.append(0)
                    ext5.append(core5[j] + mlo + mhi)
                else:
                    lo5.append(mlo)
                    ext5.append(core5[j])
            return tuple(lo5), tuple(ext5)

        lo_n, hi_n = nbrs.get(i, (None, None))
        phases.append(
            Phase(i, lo, hi, lo_n, hi_n, box(lo, hi), box(n, lo), box(0, lo), box(lo + n, hi))
        )
    return phases


def _padded5(core5, margins5):
    return tuple(c + lo + hi for c, (lo, hi) in zip(core5, margins5))


class CudaPacker:
    """The product pack/unpack path: 16-byte vectorised box kernels of libvoxmesh_sm100."""

    def _args(self, buf5, lo5, ext5):
        return _lib.ptr(buf5), _lib.i64arr(buf5.shape), _lib.i64arr(lo5), _lib.i64arr(ext5)

    def pack(self, buf5, lo5, ext5):
        import torch

        m = torch.empty(ext5, dtype=buf5.dtype, device=buf5.device)
        p, d, lo, ext = self._args(buf5, lo5, ext5)
        _lib.call("vm_box_pack", p, d, buf5.element_size(), lo, ext, _lib.ptr(m), _lib.stream_ptr())
        return m

    def unpack(self, buf5, lo5, ext5, t):
        p, d, lo, ext = self._args(buf5, lo5, ext5)
        _lib.call("vm_box_unpack", p, d, buf5.element_size(), lo, ext, _lib.ptr(t), _lib.stream_ptr())

    def unpack_add(self, buf5, lo5, ext5, t):
        p, d, lo, ext = self._args(buf5, lo5, ext5)
        _lib.call("vm_box_unpack_add", p, d, _lib.dtype_code(buf5.dtype), lo, ext, _lib.ptr(t), _lib.stream_ptr())

    def zero(self, buf5, lo5, ext5):
        p, d, lo, ext = self._args(buf5, lo5, ext5)
        _lib.call("vm_box_zero", p, d, buf5.element_size(), lo, ext, _lib.stream_ptr())


CUDA_PACKER = CudaPacker()


def _empty(like5, shape):
    import torch

    return torch.empty(shape, dtype=like5.dtype, device=like5.device)


def run_exchange(ctx, buf5, core5, margins5, nbrs, elem_bytes=None, tag=_FWD_TAG, dims_names=None, packer=None):
    """Fill the margins of the 5-D padded buffer ``buf5`` in place (forward protocol,
    halo.py:109-155).  Returns {(dim, "lo"|"hi"): "neighbor"|"zero"}."""
    pk = packer or CUDA_PACKER
    faces = {}
    for ph in plan_phases(core5, margins5, nbrs):
        name = dims_names[ph.axis_pos] if dims_names else ph.axis_pos
        sends, recvs, want = [], [], []
        if ph.lo_nbr is not None and ph.hi > 0:  # first hi interior rows travel "down"
            sends.append((ph.lo_nbr, pk.pack(buf5, *ph.send_down), (tag, name, "down")))
        if ph.hi_nbr is not None and ph.lo > 0:  # last lo interior rows travel "up"
            sends.append((ph.hi_nbr, pk.pack(buf5, *ph.send_up), (tag, name, "up")))
        if ph.lo_nbr is not None and ph.lo > 0:
            recvs.append((ph.lo_nbr, _empty(buf5, ph.recv_lo[1]), (tag, name, "up")))
            want.append(ph.recv_lo)
        if ph.hi_nbr is not None and ph.hi > 0:
            recvs.append((ph.hi_nbr, _empty(buf5, ph.recv_hi[1]), (tag, name, "down")))
            want.append(ph.recv_hi)
        got = ctx.exchange(sends, recvs) if (sends or recvs) else []
        for (lo5, ext5), t in zip(want, got):
            pk.unpack(buf5, lo5, ext5, t)
        for side, nbr, (lo5, ext5) in (("lo", ph.lo_nbr, ph.recv_lo), ("hi", ph.hi_nbr, ph.recv_hi)):
            if nbr is None and ext5[ph.axis_pos] > 0:
                pk.zero(buf5, lo5, ext5)
            faces[(name, side)] = "neighbor" if nbr is not None else "zero"
    return faces


def run_exchange_backward(ctx, buf5, core5, margins5, nbrs, tag=_BWD_TAG, dims_names=None, packer=None):
    """Adjoint (halo.py:158-194): phases reversed; each margin is sent back to the rank
    owning those voxels and added to its interior rows, low side first then high.
    In place on ``buf5``; the result is its interior."""
    pk = packer or CUDA_PACKER
    for ph in reversed(plan_phases(core5, margins5, nbrs)):
        name = dims_names[ph.axis_pos] if dims_names else ph.axis_pos
        sends, recvs, targets = [], [], []
        if ph.lo_nbr is not None and ph.lo > 0:  # margin [0,lo) goes back down
            sends.append((ph.lo_nbr, pk.pack(buf5, *ph.recv_lo), (tag, name, "down")))
        if ph.hi_nbr is not None and ph.hi > 0:  # margin [lo+n, lo+n+hi) goes back up
            sends.append((ph.hi_nbr, pk.pack(buf5, *ph.recv_hi), (tag, name, "up")))
        if ph.lo_nbr is not None and ph.hi > 0:  # first hi interior rows += from the lo neighbour
            recvs.append((ph.lo_nbr, _empty(buf5, ph.send_down[1]), (tag, name, "up")))
            targets.append(ph.send_down)
        if ph.hi_nbr is not None and ph.lo > 0:  # last lo interior rows += from the hi neighbour
            recvs.append((ph.hi_nbr, _empty(buf5, ph.send_up[1]), (tag, name, "down")))
            targets.append(ph.send_up)
        got = ctx.exchange(sends, recvs) if (sends or recvs) else []
        for (lo5, ext5), t in zip(targets, got):
            pk.unpack_add(buf5, lo5, ext5, t)


# ---------------------------------------------------------------------------
# Worker-side API (exchange_local / exchange_backward_local, halo.py:109-194)
# ---------------------------------------------------------------------------


def _spec5(block_shape, dims, halo, ctx):
    names = [n for n, _ in dims]
    if len(names) > 5:
        raise HaloError("at most 5 tensor dims are supported")
    pad = 5 - len(names)
    core5 = _pad5(block_shape)
    margins5 = [(0, 0)] * pad + [halo.margin(n) for n in names]
    nbrs = {}
    for i, (n, axis) in enumerate(dims):
        if axis is not None:
            nbrs[pad + i] = (ctx.neighbor(axis, -1), ctx.neighbor(axis, +1))
    names5 = (None,) * pad + tuple(names)
    return core5, margins5, nbrs, names5


def exchange_local(ctx, dims, halo, tag, phase_barrier, block, packer=None):
    """Worker-side forward exchange; returns the PaddedBlock (device tensor)."""
    import torch

    pk = packer or CUDA_PACKER

    core5, margins5, nbrs, names5 = _spec5(tuple(block.shape), dims, halo, ctx)
    for i, (lo, hi) in enumerate(margins5):
        if lo > core5[i] or hi > core5[i]:
            raise HaloError(
                f"margin ({lo},{hi}) on {names5[i]!r} exceeds local extent {core5[i]}; "
                "use a smaller mesh axis or a larger volume"
            )
    padded_shape = tuple(c + lo + hi for c, (lo, hi) in zip(core5, margins5))
    buf = torch.empty(padded_shape, dtype=block.dtype, device=block.device)
    inner_lo = tuple(lo for lo, _ in margins5)
    pk.unpack(buf, inner_lo, core5, block.contiguous().reshape(core5))
    faces = run_exchange(ctx, buf, core5, margins5, nbrs, tag=tag, dims_names=names5, packer=pk)
    if phase_barrier:
        pass  # stream/queue ordering replaces the per-phase barrier (halo.py:151-152)
    out_shape = tuple(e + halo.total(n) for e, (n, _) in zip(block.shape, dims))
    return PaddedBlock(buf.reshape(out_shape), halo, tuple(n for n, _ in dims), faces)


def exchange_backward_local(ctx, dims, halo, tag, phase_barrier, grad_padded, packer=None):
    """Worker-side adjoint; returns the interior gradient (device tensor)."""
    pk = packer or CUDA_PACKER

    g = grad_padded.data if isinstance(grad_padded, PaddedBlock) else grad_padded
    names = [n for n, _ in dims]
    core = tuple(e - halo.total(n) for e, n in zip(g.shape, names))
    for e, n in zip(core, names):
        if e <= 0:
            lo, hi = halo.margin(n)
            raise HaloError(f"gradient block extent {e + lo + hi} too small for margins ({lo},{hi}) on {n!r}")
    core5, margins5, nbrs, names5 = _spec5(core, dims, halo, ctx)
    buf = g.contiguous().clone().reshape(_padded5(core5, margins5))
    run_exchange_backward(ctx, buf, core5, margins5, nbrs, tag=tag, dims_names=names5, packer=pk)
    inner_lo = tuple(lo for lo, _ in margins5)
    return pk.pack(buf, inner_lo, core5).reshape(core)


def exchange_byte_count(spec, layout, mesh, halo, direction="forward"):
    """Analytic bytes sent by all workers in one exchange (halo.py:197-229)."""
    if direction not in ("forward", "backward"):
        raise ValueError(f"direction must be forward|backward, got {direction!r}")
    layout.validate(spec, mesh)
    cur0 = list(local_shape(spec, layout, mesh))
    total = 0
    for coord in mesh.coords:
        cur = list(cur0)
        for i, name in enumerate(spec.names):
            lo, hi = halo.margin(name)
            if lo == 0 and hi == 0:
                continue
            axis = layout.axis_for(name)
            if axis is not None and mesh.axis_size(axis) > 1:
                area = 1
                for j, e in enumerate(cur):
                    if j != i:
                        area *= e
                c = coord[mesh.axis_index[axis]]
                down, up = (hi, lo) if direction == "forward" else (lo, hi)
                total += down * area if c > 0 else 0
                total += up * area if c < mesh.axis_size(axis) - 1 else 0
            cur[i] += lo + hi
    return total * spec.dtype.itemsize


def halo_exchange(x: ShardedTensor, halo, phase_barrier=True):
    """Collective forward exchange; one PaddedBlock per rank (None for remote ranks)."""
    dims = dim_axes(x.spec, x.layout)
    return x.mesh.run(exchange_local, dims, halo, _FWD_TAG, phase_barrier, per_worker=(x.blocks,))


def halo_exchange_backward(grad_padded, x_spec, layout, mesh, halo, phase_barrier=True):
    """Collective adjoint; returns the interior gradient as a ShardedTensor."""
    import torch

    dims = dim_axes(x_spec, layout)
    base = local_shape(x_spec, layout, mesh)
    expected = tuple(e + halo.total(n) for e, n in zip(base, x_spec.names))
    arrays = []
    for r, g in enumerate(grad_padded):
        if g is None:
            arrays.append(None)
            continue
        arr = g.data if isinstance(g, PaddedBlock) else g
        if not isinstance(arr, torch.Tensor):
            arr = torch.as_tensor(arr).to(mesh.device_of(r))
        if tuple(arr.shape) != expected:
            raise HaloError(
                f"gradient block shape {tuple(arr.shape)} does not match padded shape {expected} "
                f"for margins {halo.margins}"
            )
        if arr.dtype != torch_dtype(x_spec.dtype):
            arr = arr.to(torch_dtype(x_spec.dtype))
        arrays.append(arr)
    blocks = mesh.run(exchange_backward_local, dims, halo, _BWD_TAG, phase_barrier, per_worker=(arrays,))
    return ShardedTensor(x_spec, layout, mesh, blocks)


# ---------------------------------------------------------------------------
# The U-Net step's halo: channel-blocked padded slabs [B][CG][D+2][H+2][W+2][8]
# ---------------------------------------------------------------------------


class CudaSlabKernels:
    """Per-phase pack / unpack of a slab's faces, one launch for every (sample, channel
    group) and both sides (vm_halo_slab_pack / _unpack, csrc/halo.cu)."""

    def _geom(self, s):
        return _lib.dtype_code(s.dtype), s.p(), s.bstride, s.B, s.C, s.D, s.H, s.W

    def face_bytes(self, s, axis):
        return int(_lib.load().vm_halo_slab_face_bytes(_lib.dtype_code(s.dtype), s.B, s.C, s.D, s.H, s.W, axis))

    def pack(self, s, axis, down, up):
        import torch

        n = self.face_bytes(s, axis) // s.storage.element_size()
        md = torch.empty(n, dtype=s.dtype, device=s.storage.device) if down else None
        mu = torch.empty(n, dtype=s.dtype, device=s.storage.device) if up else None
        _lib.call("vm_halo_slab_pack", *self._geom(s), axis, _lib.ptr(md), _lib.ptr(mu), _lib.stream_ptr())
        return md, mu

    def like(self, s, axis):
        import torch

        return torch.empty(self.face_bytes(s, axis) // s.storage.element_size(), dtype=s.dtype,
                           device=s.storage.device)

    def unpack(self, s, axis, from_lo, from_hi):
        _lib.call("vm_halo_slab_unpack", *self._geom(s), axis, _lib.ptr(from_lo), _lib.ptr(from_hi),
                  _lib.stream_ptr())

    def zero(self, s, nbr6):
        _lib.call("vm_halo_slab_zero", _lib.dtype_code(s.dtype), s.p(), s.bstride, s.B, s.C, s.D, s.H, s.W,
                  (ctypes.c_int * 6)(*nbr6), _lib.stream_ptr())


class TorchSlabKernels:
    """Tensor-slicing restatement of CudaSlabKernels (same face boxes and message layout
    [B][CG][n1][n2][8]), so the slab protocol and its transports run on CPU (gloo tests)."""

    @staticmethod
    def view(s):
        Dp, Hp, Wp = s.D + 2, s.H + 2, s.W + 2
        return s.storage.as_strided((s.B, s.CG, Dp, Hp, Wp, 8), (s.bstride, Dp * Hp * Wp * 8, Hp * Wp * 8, Wp * 8, 8, 1),
                                    s.offset)

    @staticmethod
    def _box(s, axis, pos, full=False):
        if axis == 0:
            return (slice(None), slice(None), pos, slice(None) if full else slice(1, s.H + 1),
                    slice(None) if full else slice(1, s.W + 1))
        if axis == 1:
            return slice(None), slice(None), slice(None), pos, slice(None) if full else slice(1, s.W + 1)
        return slice(None), slice(None), slice(None), slice(None), pos

    def face_bytes(self, s, axis):
        return self.view(s)[self._box(s, axis, 1)].numel() * s.storage.element_size()

    def pack(self, s, axis, down, up):
        v = self.view(s)
        n = (s.D, s.H, s.W)[axis]
        md = v[self._box(s, axis, 1)].contiguous().reshape(-1) if down else None
        mu = v[self._box(s, axis, n)].contiguous().reshape(-1) if up else None
        return md, mu

    def like(self, s, axis):
        import torch

        return torch.empty(self.face_bytes(s, axis) // s.storage.element_size(), dtype=s.dtype,
                           device=s.storage.device)

    def unpack(self, s, axis, from_lo, from_hi):
        v = self.view(s)
        n = (s.D, s.H, s.W)[axis]
        for pos, m in ((0, from_lo), (n + 1, from_hi)):
            if m is not None:
                dst = v[self._box(s, axis, pos)]
                dst.copy_(m.reshape(dst.shape))

    def zero(self, s, nbr6):
        v = self.view(s)
        for a in range(3):
            n = (s.D, s.H, s.W)[a]
            for side, pos in ((0, 0), (1, n + 1)):
                if nbr6[2 * a + side] >= 0:
                    v[self._box(s, a, pos, full=True)] = 0


class SlabHalo:
    """Forward halo of the step's slabs (the 3-phase protocol of halo.py:109-155, margin 1).

    ``nbr6`` = lo/hi neighbour ranks of the D, H, W dims (-1 at a global boundary).  Two
    transports, same bytes and the same messages:

    * ``comm`` (an ncclComm_t): one C call per slab, vm_halo_slab_fwd — pack, NCCL group,
      unpack per phase on the caller's stream, capturable in a CUDA graph (spmd over NCCL);
    * ``ctx`` (a mesh WorkerContext): the phases driven from the host around
      ``ctx.exchange`` (threads mesh on one GPU, gloo on CPU), with ``kernels`` doing the
      per-phase pack / unpack (CudaSlabKernels, or TorchSlabKernels on CPU).
    """

    def __init__(self, nbr6, ctx=None, comm=None, kernels=None, nbr26=None):
        self.nbr6 = [int(n) for n in nbr6]
        self.ctx, self.comm = ctx, comm
        self.kernels = kernels or CudaSlabKernels()
        self.ws = None
        self._sent = ctypes.c_longlong(0)
        # one-phase exchange (vm_halo_slab_fwd26) on meshes that split more than one spatial dim:
        # one pack / NCCL group / unpack per exchange instead of one per dim (VOXMESH_HALO_PHASES
        # = 3 forces the sequential protocol, = 1 the one-phase one on any mesh)
        split = sum(1 for a in range(3) if self.nbr6[2 * a] >= 0 or self.nbr6[2 * a + 1] >= 0)
        phases = os.environ.get("VOXMESH_HALO_PHASES", "")
        self.nbr26 = None
        if nbr26 is not None and (phases == "1" or (split > 1 and phases != "3")):
            self.nbr26 = [int(n) for n in nbr26]

    @property
    def active(self):
        return any(n >= 0 for n in self.nbr6)

    def reserve(self, slabs):
        """Preallocate the NCCL message scratch for the largest of ``slabs``."""
        if self.comm is None:
            return
        import torch

        fn = "vm_halo_slab_ws_bytes26" if self.nbr26 is not None else "vm_halo_slab_ws_bytes"
        need = max(int(_lib.call_size(fn, _lib.dtype_code(s.dtype), s.B, s.C, s.D, s.H, s.W)) for s in slabs)
        dev = slabs[0].storage.device
        self.ws = torch.empty(need // 4 + 64, dtype=torch.float32, device=dev)
        self.ws_bytes = self.ws.numel() * 4

    def bytes_sent(self):
        return int(self._sent.value)

    def forward(self, s, tag=_FWD_TAG):
        if not self.active:
            return
        if self.comm is not None and self.nbr26 is not None:
            _lib.call("vm_halo_slab_fwd26", ctypes.c_void_p(self.comm), _lib.dtype_code(s.dtype), s.p(), s.bstride,
                      s.B, s.C, s.D, s.H, s.W, (ctypes.c_int * 26)(*self.nbr26), _lib.ptr(self.ws), self.ws_bytes,
                      ctypes.byref(self._sent), _lib.stream_ptr())
            if self.ctx is not None:
                self.ctx.counters["p2p_bytes"] = self.bytes_sent()
            return
        if self.comm is not None:
            _lib.call("vm_halo_slab_fwd", ctypes.c_void_p(self.comm), _lib.dtype_code(s.dtype), s.p(), s.bstride, s.B,
                      s.C, s.D, s.H, s.W, (ctypes.c_int * 6)(*self.nbr6), _lib.ptr(self.ws), self.ws_bytes,
                      ctypes.byref(self._sent), _lib.stream_ptr())
            if self.ctx is not None:
                self.ctx.counters["p2p_bytes"] = self.bytes_sent()
            return
        k = self.kernels
        for a in range(3):
            lo, hi = self.nbr6[2 * a], self.nbr6[2 * a + 1]
            if lo < 0 and hi < 0:
                continue
            down, up = k.pack(s, a, lo >= 0, hi >= 0)
            sends, recvs = [], []
            if lo >= 0:
                sends.append((lo, down, (tag, a, "down")))
            if hi >= 0:
                sends.append((hi, up, (tag, a, "up")))
            if lo >= 0:
                recvs.append((lo, k.like(s, a), (tag, a, "up")))
            if hi >= 0:
                recvs.append((hi, k.like(s, a), (tag, a, "down")))
            got = iter(self.ctx.exchange(sends, recvs))
            k.unpack(s, a, next(got) if lo >= 0 else None, next(got) if hi >= 0 else None)

    def zero(self, s):
        """Zero the margins this halo wrote (a gradient slab before its weight gradient)."""
        if self.active:
            self.kernels.zero(s, self.nbr6)


def directions26():
    """Offsets (sd, sh, sw) in {-1,0,1}^3 without the center, in the order of vm_halo_slab_fwd26's
    nbr26 (lexicographic; the opposite of direction k is 25 - k)."""
    return [(t // 9 - 1, (t // 3) % 3 - 1, t % 3 - 1) for t in range(27) if t != 13]


def nbr26_of(nbr6, rank_at=None):
    """Face, edge and corner neighbours from the face neighbours ``nbr6``: direction s exists
    when every nonzero component has a neighbour on that side; its rank is ``rank_at(s)``
    (the mesh coordinate + s), or, with ``rank_at`` None, the single rank all face neighbours
    share (the periodic single-GPU emulation, every neighbour = this rank)."""
    out = []
    for s in directions26():
        ok = all(si == 0 or nbr6[2 * a + (si > 0)] >= 0 for a, si in enumerate(s))
        if not ok:
            out.append(-1)
        elif rank_at is not None:
            out.append(int(rank_at(s)))
        else:
            ranks = {n for n in nbr6 if n >= 0}
            if len(ranks) != 1:
                raise HaloError("nbr26_of: diagonal ranks need rank_at unless all neighbours are one rank")
            out.append(ranks.pop())
    return out


class HaloLinkC(ctypes.Structure):
    """vm_halo_link (include/vm_api.h)."""

    _fields_ = [("push_lo", ctypes.c_void_p), ("push_hi", ctypes.c_void_p), ("lo_flag", ctypes.c_void_p),
                ("hi_flag", ctypes.c_void_p), ("counter", ctypes.c_void_p), ("wait_own", ctypes.c_void_p),
                ("wait_lo", ctypes.c_int), ("wait_hi", ctypes.c_int), ("epoch", ctypes.c_void_p)]

    @classmethod
    def of(cls, push=None, wait=None):
        if push is None and wait is None:
            return None
        f = dict(push or {})
        for k, v in (wait or {}).items():
            f[k] = v
        return cls(**{k: v for k, v in f.items() if v is not None})


class PeerDepthHalo:
    """Depth-only halo through peer memory (vm_halo_depth_push): no NCCL, no pack / unpack.

    Each exchange is ONE launch that pushes this rank's first / last interior depth layers
    into the lo / hi neighbours' margin layers (NVLink P2P stores through CUDA-IPC mappings of
    the neighbours' slabs), publishes the step epoch into their flag words and waits for its
    own margins.  Exchanges are numbered in program order within a step (the same on every
    rank: every rank runs the same static step program); ``begin_step`` bumps the device
    epoch and restarts the numbering, so a captured step graph replays correctly.

    ``peers=None``: every neighbour is this rank itself (the periodic single-GPU emulation of a
    split: the same launches and bytes, local HBM instead of NVLink).  Otherwise call
    :meth:`connect` with the exchanged slabs (spmd over NCCL: handles are swapped with
    ``torch.distributed.all_gather_object``).
    """

    NSLOT = 512

    def __init__(self, nbr6, device, self_peers=True):
        import torch

        if any(n >= 0 for n in nbr6[2:]):
            raise HaloError("peer-memory halo: only a depth split (x axis) is supported")
        self.nbr6 = [int(n) for n in nbr6]
        self.comm = None
        self.self_peers = self_peers
        self.state = torch.zeros(8 + 3 * self.NSLOT, dtype=torch.int32, device=device)
        self.peer_state = (self.state.data_ptr(), self.state.data_ptr()) if self_peers else (None, None)
        self.peer_slab = {}  # own slab pointer -> (lo neighbour's, hi neighbour's)
        self._slot = 0
        self._pending = {}
        self._sent = 0
        # the weight-gradient kernels never read a depth margin layer of gy, so they may run
        # while this transport fills them (UNetStep overlaps wgrad with exchange + dgrad)
        self.wgrad_safe = True

    @property
    def active(self):
        return self.nbr6[0] >= 0 or self.nbr6[1] >= 0

    def reserve(self, slabs):
        pass

    def bytes_sent(self):
        return self._sent

    def connect(self, slabs, group=None):
        """Map the neighbours' copies of ``slabs`` (same program order on every rank) and
        their flag words through CUDA IPC."""
        import torch.distributed as dist

        def rec(ptr):
            h = ctypes.create_string_buffer(64)
            off = ctypes.c_int64(0)
            _lib.call("vm_ipc_handle", ctypes.c_void_p(ptr), ctypes.addressof(h), ctypes.addressof(off))
            return (h.raw, int(off.value))

        mine = [rec(self.state.data_ptr())] + [rec(s.ptr) for s in slabs]
        world = [None] * dist.get_world_size(group)
        dist.all_gather_object(world, mine, group=group)

        def open_(r):
            out = []
            for h, off in world[r]:
                base = ctypes.c_void_p(0)
                hb = ctypes.create_string_buffer(h, 64)
                _lib.call("vm_ipc_open", ctypes.addressof(hb), ctypes.addressof(base))
                out.append(int(base.value) + off)
            return out

        err = None
        try:
            lo = open_(self.nbr6[0]) if self.nbr6[0] >= 0 else None
            hi = open_(self.nbr6[1]) if self.nbr6[1] >= 0 else None
        except Exception as e:  # noqa: BLE001 - decided collectively below
            err = e
        import torch

        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=self.state.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)  # every rank takes the same transport
        if not int(ok.item()):
            raise HaloError(f"peer-memory halo: CUDA-IPC mapping failed on some rank ({err or 'elsewhere'})")
        self.peer_state = (lo[0] if lo else None, hi[0] if hi else None)
        for i, s in enumerate(slabs):
            self.peer_slab[s.ptr] = (lo[1 + i] if lo else None, hi[1 + i] if hi else None)
        self.self_peers = False

    def begin_step(self):
        self._slot = 0
        self._pending = {}
        _lib.call("vm_halo_epoch_bump", _lib.ptr(self.state), _lib.stream_ptr())

    def forward(self, s, tag=_FWD_TAG):
        if not self.active:
            return
        slot = self._next_slot()
        lo_n, hi_n = self.nbr6[0] >= 0, self.nbr6[1] >= 0
        if self.self_peers:
            lo_p, hi_p = s.ptr, s.ptr
        else:
            lo_p, hi_p = self.peer_slab[s.ptr]
        base = self.state.data_ptr()
        own = base + 4 * (8 + 2 * slot)
        lo_flag = self.peer_state[0] + 4 * (8 + 2 * slot + 1) if lo_n else None
        hi_flag = self.peer_state[1] + 4 * (8 + 2 * slot) if hi_n else None
        counter = base + 4 * (8 + 2 * self.NSLOT + slot)
        vp = ctypes.c_void_p
        _lib.call("vm_halo_depth_push", _lib.dtype_code(s.dtype), s.p(), s.bstride, s.B, s.C, s.D, s.H, s.W,
                  vp(lo_p) if lo_n else None, vp(hi_p) if hi_n else None, vp(lo_flag) if lo_n else None,
                  vp(hi_flag) if hi_n else None, vp(own), vp(counter), vp(base), _lib.stream_ptr())
        self._sent += s.B * s.CG * 8 * s.H * s.W * s.storage.element_size() * (lo_n + hi_n)

    def check(self):
        """Raise if an exchange of this transport timed out waiting for a neighbour (host sync)."""
        err = int(self.state[1].item())
        if err:
            raise HaloError(f"peer-memory halo: a neighbour's signal did not arrive (epoch {err})")

    def zero(self, s):
        """Zero the exchanged depth margins (the serial path of a transport user whose weight
        gradient reads them; the tensor-core wgrad never does)."""
        if self.active:
            _lib.call("vm_halo_slab_zero", _lib.dtype_code(s.dtype), s.p(), s.bstride, s.B, s.C, s.D, s.H, s.W,
                      (ctypes.c_int * 6)(*self.nbr6), _lib.stream_ptr())

    # ---- fused exchanges (the producer conv pushes, the consumer conv waits) ------------
    def reserve_push(self, y):
        """Producer side: the next exchange slot for slab ``y``, whose producer kernel pushes
        its boundary layers itself; returns the vm_halo_link fields of that push."""
        if not self.active:
            return None
        slot = self._next_slot()
        self._pending[y.ptr] = slot
        lo_n, hi_n = self.nbr6[0] >= 0, self.nbr6[1] >= 0
        lo_p, hi_p = (y.ptr, y.ptr) if self.self_peers else self.peer_slab[y.ptr]
        base = self.state.data_ptr()
        self._sent += y.B * y.CG * 8 * y.H * y.W * y.storage.element_size() * (lo_n + hi_n)
        return dict(push_lo=lo_p if lo_n else None, push_hi=hi_p if hi_n else None,
                    lo_flag=self.peer_state[0] + 4 * (8 + 2 * slot + 1) if lo_n else None,
                    hi_flag=self.peer_state[1] + 4 * (8 + 2 * slot) if hi_n else None,
                    counter=base + 4 * (8 + 2 * self.NSLOT + slot), epoch=base)

    def consume(self, s):
        """Consumer side of a conv input: the slot a fused producer pushed ``s`` under (the
        consumer kernel waits on it: vm_halo_link wait fields), or None after a standalone
        push here (vm_halo_depth_push, which waits itself)."""
        slot = self._pending.pop(s.ptr, None)
        if slot is None:
            self.forward(s)
            return None
        base = self.state.data_ptr()
        return dict(wait_own=base + 4 * (8 + 2 * slot), wait_lo=int(self.nbr6[0] >= 0),
                    wait_hi=int(self.nbr6[1] >= 0), epoch=base)

    def _next_slot(self):
        slot = self._slot
        if slot >= self.NSLOT:
            raise HaloError(f"peer-memory halo: more than {self.NSLOT} exchanges in one step")
        self._slot += 1
        return slot


def nccl_comm_ptr(group=None):
    """The ncclComm_t behind a torch.distributed NCCL process group (initialised eagerly by a
    one-element all-reduce when torch created it lazily)."""
    import torch
    import torch.distributed as dist

    g = group if group is not None else dist.group.WORLD
    backend = g._get_backend(torch.device("cuda"))
    try:
        ptr = int(backend._comm_ptr())
    except Exception:  # noqa: BLE001 - lazily created communicator
        ptr = 0
    if not ptr:
        t = torch.zeros(1, device="cuda")
        dist.all_reduce(t, group=g)
        torch.cuda.synchronize()
        ptr = int(backend._comm_ptr())
    _lib.call("vm_nccl_bind")
    return ptr


def nccl_comm_of(ctx):
    """The world NCCL communicator of an spmd mesh over NCCL, else None (threads / gloo)."""
    if ctx is None or ctx.mesh.backend != "spmd" or ctx.device.type != "cuda":
        return None
    import torch.distributed as dist

    if dist.get_backend() != "nccl":
        return None
    return nccl_comm_ptr()


def nccl_second_comm(ctx):
    """A second NCCL communicator over all ranks (the bucketed weight-gradient all-reduce runs
    on its own stream and communicator, concurrently with the halo's), cached per mesh."""
    if nccl_comm_of(ctx) is None:
        return None
    mesh = ctx.mesh
    if getattr(mesh, "_ar_comm", None) is None:
        import torch.distributed as dist

        mesh._ar_group = dist.new_group(backend="nccl")
        mesh._ar_comm = nccl_comm_ptr(mesh._ar_group)
    return mesh._ar_comm
