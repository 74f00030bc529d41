"""The per-GPU U-Net train step on channel-blocked padded slabs (the hot path).

Replaces the reference's per-worker graph interpreter (``unet.run_forward_local``
/ ``run_backward_local``, unet.py:331-442) and ``training._train_step``
(training.py:330-343) with a static program over pre-allocated device buffers:

* every activation lives in a slab ``[B][ceil(C/8)][D+2][H+2][W+2][8]`` (bf16 or
  fp32); producers write interiors, the halo exchange writes margins, global
  boundary margins stay zero (no re-padding, halo.py:148);
* conv + bias + ReLU is one kernel (the tape keeps the post-ReLU output only:
  y>0 <=> x>0, ops.py:186-187); decoder concat [up, skip] is zero-copy when the
  upsampled channel count is a multiple of 8 (the encoder's last conv writes
  straight into the skip half of the concat slab);
* backward: wgrad(x, g) -> [halo(g)] -> dgrad = forward conv of g with flipped,
  transposed taps, whose epilogue applies the previous layer's ReLU mask;
  maxpool / upsample backward fuse the fan-out add and the mask;
* head 1x1x1 conv + softmax + Dice/CE statistics in one kernel; statistics and
  weight gradients are summed over the mesh (ctx.all_reduce_sum -> NCCL
  all_reduce in spmd mode); SGD with momentum + non-finite skip in one launch.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .errors import GraphBuildError, VoxmeshError
from .halo import HaloLinkC, PeerDepthHalo, SlabHalo, nbr26_of, nccl_comm_of, nccl_second_comm

_DT = {torch.bfloat16: _lib.VM_BF16, torch.float32: _lib.VM_F32}


class Slab:
    """Channel-blocked padded buffer; may be a channel-group window of a wider slab."""

    TAIL = 64 * 1024  # elements

    def __init__(self, B, C, D, H, W, dtype, device, parent=None, cg0=0):
        self.B, self.C, self.D, self.H, self.W = B, C, D, H, W
        self.CG = (C + 7) // 8
        self.dtype = dtype
        self.plane = (D + 2) * (H + 2) * (W + 2) * 8
        if parent is None:
            # + tail pad: the tensor-core kernels bulk-copy whole row runs and may read
            # (and discard) up to a few thousand rows past the last plane
            self.storage = torch.zeros(B * self.CG * self.plane + self.TAIL, dtype=dtype, device=device)
            self.bstride = self.CG * self.plane
            self.offset = 0
        else:
            assert parent.plane == self.plane and parent.dtype == dtype
            self.storage = parent.storage
            self.bstride = parent.bstride
            self.offset = parent.offset + cg0 * self.plane
        self.parent = parent

    @property
    def ptr(self):
        return self.storage.data_ptr() + self.offset * self.storage.element_size()

    def p(self):
        return _lib.ctypes.c_void_p(self.ptr)

    def view5(self, b):
        """[CG, D+2, H+2, W+2, 8] view of sample b (for halo box kernels)."""
        return self.storage.as_strided(
            (self.CG, self.D + 2, self.H + 2, self.W + 2, 8),
            (self.plane, (self.H + 2) * (self.W + 2) * 8, (self.W + 2) * 8, 8, 1),
            self.offset + b * self.bstride,
        )

    def interior(self):
        """Dense [B, D, H, W, C] fp32 copy of the interior (test/debug helper)."""
        out = torch.empty((self.B, self.D, self.H, self.W, self.C), dtype=torch.float32, device=self.storage.device)
        _lib.call(
            "vm_slab_to_dense", self.p(), _DT[self.dtype], self.bstride, _lib.ptr(out), _lib.VM_F32,
            self.B, self.C, self.D, self.H, self.W, 1, _lib.stream_ptr(),
        )
        return out


class ConvLayer:
    def __init__(self, node, index, D, H, W):
        self.node, self.index = node, index
        self.k, self.cin, self.cout = node.k, node.c_in, node.c_out
        self.D, self.H, self.W = D, H, W
        self.nk = self.k ** 3 * self.cin * self.cout


class UNetStep:
    """Static train-step program for one rank's block.

    ``params`` is the reference-format dict {conv id: {"kernel": [k,k,k,ci,co], "bias": [co]}}.
    ``ctx`` (a mesh WorkerContext) supplies neighbours, halo transport and
    all-reduce; ``None`` means a single unpartitioned rank.
    """

    def __init__(self, graph, params, batch=1, ctx=None, device=None, dtype=torch.bfloat16,
                 conv_impl="tc", lr=0.003, momentum=0.9, loss_weights=(0.9, 0.1),
                 dice_classes=(1, 2), clamp=1e-12, global_batch=None, global_shape=None, local_shape=None):
        cfg = graph.config
        if cfg.kernel != 3:
            raise GraphBuildError(f"the slab step supports 3x3x3 convolutions, got k={cfg.kernel}")
        self.graph, self.cfg, self.ctx = graph, cfg, ctx
        self.device = torch.device(device) if device is not None else (ctx.device if ctx else torch.device("cuda"))
        if self.device.type != "cuda":
            raise VoxmeshError("the step program needs a CUDA device (no CPU fallback)")
        _lib.load()
        self.dtype, self.dt = dtype, _DT[dtype]
        self.conv_impl = conv_impl if dtype == torch.bfloat16 else "simt"
        self.B = batch
        self.lr, self.mu = float(lr), float(momentum)
        self.w_dice, self.w_ce = loss_weights
        self.dice_mask = sum(1 << k for k in dice_classes)
        self.clamp = clamp
        self.keep_probs = False
        self.probs = None
        self.keep_pred = False  # evaluation: u8 argmax class per voxel (training.py:355)
        self.pred = None
        # mesh axes the loss statistics are summed over: None = all (training.py:337); the
        # evaluation's per-sample statistics use the spatial axes only (training.py:353-354)
        self.stats_axes = None
        self.ncls = cfg.num_classes
        # local extents per spatial dim (x->D, y->H, z->W)
        layout, mesh = graph.layout, graph.mesh
        self.div = [1, 1, 1]
        self.nbrs = {}
        for i, d in enumerate(("x", "y", "z")):
            a = layout.axis_for(d) if layout is not None else None
            if a is not None and mesh is not None:
                self.div[i] = mesh.axis_size(a)
                if ctx is not None:
                    self.nbrs[1 + i] = (ctx.neighbor(a, -1), ctx.neighbor(a, +1))
        self.has_halo = any(lo is not None or hi is not None for lo, hi in self.nbrs.values())
        nbr6 = [-1] * 6
        for i in range(3):
            lo, hi = self.nbrs.get(1 + i, (None, None))
            nbr6[2 * i], nbr6[2 * i + 1] = (-1 if lo is None else lo), (-1 if hi is None else hi)
        # the halo transport: NCCL through the C ABI when the mesh is spmd over NCCL (one C call
        # per slab, graph-capturable), else host-driven phases around ctx.exchange (threads)
        comm = nccl_comm_of(ctx)
        self.halo = SlabHalo(nbr6, ctx=ctx, comm=comm,
                             nbr26=self._nbr26(ctx, layout, nbr6) if comm is not None else None)
        self.comm = self.halo.comm  # NCCL communicator of the step's collectives (None: ctx's)
        self.ar_comm = nccl_second_comm(ctx)  # bucketed weight-gradient all-reduce
        # overlap the exchange with the conv's interior planes: only the depth axis is split
        # (cfg3); the interior output planes [1, D-1) read no margin plane
        self.overlap_halo = True
        self.overlap_min_planes = 32  # tools/halo_ab.py: the boundary launches cost more below
        self.halo_sm_reserve = 8  # SMs the interior conv leaves to the overlapped exchange
        self.fuse_halo = True  # peer transport: producer convs push their boundary layers themselves
        self.defer_finalize = True  # wgrad K-split finalize on its own stream (two workspaces)
        self.bucket_bytes = 16 << 20
        bdiv = mesh.axis_size(layout.axis_for("batch")) if (layout is not None and layout.axis_for("batch")) else 1
        self.global_batch = global_batch or batch * bdiv
        E = cfg.input_extent
        self.global_shape = tuple(global_shape) if global_shape else (E, E, E)
        # local block of the level-0 volume; deeper levels scale by level_extent / E
        self.local_shape = tuple(local_shape) if local_shape else tuple(
            g // d for g, d in zip(self.global_shape, self.div))
        self.total_voxels = float(self.global_batch * int(np.prod(self.global_shape)))
        self._rec = None
        self.overlap_wgrad = True  # weight gradients on a side stream, concurrent with dgrad
        # programmatic dependent launch (the next kernel's CTAs are scheduled and set up while
        # the previous one drains).  Forward: trigger at kernel start.  Backward: trigger at CTA
        # exit only — CTAs parked early at the dependency wait would take SMs from the
        # side-stream wgrad (measured: early 3.22 ms, late 3.12 ms, off 3.17 ms per step)
        self.first_layer_c1 = True  # Cin = 1 convs through the im2col kernels (vm_conv3d_*_c1)
        self.pdl_forward = 1  # 0 off, 1 trigger at kernel start, 2 trigger at CTA exit
        self.pdl_backward = 2
        self._build_buffers(params)
        self._reserve_halo()

    # ------------------------------------------------------------------ setup
    def _ext(self, nid):
        shrink = self.cfg.input_extent // self.graph.level_extents[nid]
        return tuple(n // shrink for n in self.local_shape)

    def _slab(self, C, ext, parent=None, cg0=0):
        return Slab(self.B, C, *ext, self.dtype, self.device, parent, cg0)

    def _build_buffers(self, params):
        g = self.graph
        dev = self.device
        convs = g.conv_nodes
        self.layers = []
        offs = [0]
        for i, n in enumerate(convs):
            L = ConvLayer(n, i, *self._ext(n.id))
            self.layers.append(L)
            offs.append(offs[-1] + L.nk + n.c_out)
        self.by_id = {L.node.id: L for L in self.layers}
        total = offs[-1]
        self.offsets_host = offs
        self.offsets = torch.tensor(offs, dtype=torch.int64, device=dev)
        self.max_layer = max(b - a for a, b in zip(offs, offs[1:]))
        self.params = torch.zeros(total, dtype=torch.float32, device=dev)
        self.moments = torch.zeros(total, dtype=torch.float32, device=dev)
        self.grads = torch.zeros(total, dtype=torch.float32, device=dev)
        self.skip_flags = torch.zeros(len(self.layers), dtype=torch.int32, device=dev)
        host = np.zeros(total, dtype=np.float32)
        for L, a in zip(self.layers, offs):
            p = params[L.node.id]
            host[a : a + L.nk] = np.asarray(p["kernel"], dtype=np.float32).reshape(-1)
            host[a + L.nk : a + L.nk + L.cout] = np.asarray(p["bias"], dtype=np.float32)
        self.params.copy_(torch.from_numpy(host))
        for L, a in zip(self.layers, offs):
            L.w = self.params[a : a + L.nk]
            L.b = self.params[a + L.nk : a + L.nk + L.cout]
            L.gw = self.grads[a : a + L.nk]
            L.gb = self.grads[a + L.nk : a + L.nk + L.cout]
            if L.k == 3:
                if self.conv_impl == "tc":
                    nbytes = int(_lib.call_size("vm_packed_weights_bytes", L.cin, L.cout))
                    L.wp = torch.empty(nbytes // 2, dtype=torch.bfloat16, device=dev)
                    L.wpt = torch.empty(int(_lib.call_size("vm_packed_weights_bytes", L.cout, L.cin)) // 2,
                                        dtype=torch.bfloat16, device=dev)
                else:
                    L.wt = torch.empty(L.nk, dtype=torch.float32, device=dev)
                ws_fn = "vm_conv3d_wgrad_tc_ws" if self.conv_impl == "tc" else "vm_conv3d_wgrad_simt_ws"
                L.ws_bytes = int(_lib.call_size(ws_fn, self.B, L.cin, L.cout, L.D, L.H, L.W))
                # single-channel first conv: im2col tcgen05 kernels (27 taps as K) on a compact
                # copy of the input (no halo: a partitioned rank keeps the slab path, whose
                # margins receive the neighbours' faces)
                L.c1 = (self.conv_impl == "tc" and self.first_layer_c1 and not self.has_halo and L.cin == 1
                        and L.cout <= 32)
                if L.c1:
                    L.ws_bytes = max(L.ws_bytes, int(_lib.call_size("vm_conv3d_wgrad_c1_ws", self.B, L.cout,
                                                                    L.D, L.H, L.W)))
        self.wgrad_ws = torch.empty(max([L.ws_bytes for L in self.layers if L.k == 3] + [16]) // 4 + 4,
                                    dtype=torch.float32, device=dev)
        # second workspace: the K-split finalize of one layer runs on its own stream while the
        # next layer's weight gradient fills the other workspace (defer_finalize)
        self.wgrad_ws2 = torch.empty_like(self.wgrad_ws) if self.conv_impl == "tc" else None
        # split-K scratch of the general forward/dgrad kernel (deep levels); zeroed once, its
        # tile counters return to zero after every launch.  Main stream only.
        conv_ws = [16]
        if self.conv_impl == "tc":
            for L in self.layers:
                if L.k == 3:
                    for ci, co in ((L.cin, L.cout), (L.cout, L.cin)):
                        conv_ws.append(int(_lib.call_size("vm_conv3d_fwd_tc_ws_bytes", self.B, ci, co, L.D, L.H, L.W)))
        self.conv_ws_bytes = max(conv_ws)
        self.conv_ws = torch.zeros(self.conv_ws_bytes // 4 + 64, dtype=torch.float32, device=dev)

        # activation slabs -------------------------------------------------
        self.out = {}  # node id -> Slab holding that node's output (relu shares its conv's slab)
        nodes = g.nodes
        consumers = {}
        for n in nodes:
            for inp in n.inputs:
                consumers.setdefault(inp, []).append(n)
        self.consumers = consumers
        cfg = self.cfg
        e0 = self._ext(nodes[0].id)
        self.x_in = self._slab(cfg.in_channels, e0)
        self.out["input"] = self.x_in
        # compact single-channel copy of the input for the Cin = 1 im2col convs
        self.x1 = None
        # the 8-channel input slab is only written when a consumer still reads it
        self.input_slab_needed = not all(
            self.by_id[n.id].c1 for n in g.nodes if n.op == "conv" and n.k == 3 and n.inputs[0] == "input")
        if any(getattr(L, "c1", False) for L in self.layers):
            self.x1 = torch.zeros(self.B * (e0[0] + 2) * (e0[1] + 2) * (e0[2] + 2), dtype=torch.bfloat16,
                                  device=dev)
        self.cat_parts = {}
        # concat slabs first, so skip producers can write into them
        for n in nodes:
            if n.op == "concat":
                up_id, skip_id = n.inputs
                c_up = self.graph.node(up_id).c_out
                cat = self._slab(n.c_out, self._ext(n.id))
                self.out[n.id] = cat
                aligned = c_up % 8 == 0
                self.cat_parts[n.id] = (c_up, aligned)
                if aligned:
                    self.out[up_id] = self._slab(c_up, self._ext(n.id), parent=cat, cg0=0)
                    skip_c = n.c_out - c_up
                    self.out[skip_id] = self._slab(skip_c, self._ext(n.id), parent=cat, cg0=c_up // 8)
        for n in nodes:
            if n.id in self.out:
                continue
            if n.op == "conv" and n.k == 3:
                relu = next(c for c in consumers[n.id] if c.op == "relu")
                if relu.id in self.out:  # skip source written into the concat slab
                    self.out[n.id] = self.out[relu.id]
                else:
                    self.out[n.id] = self._slab(n.c_out, self._ext(n.id))
                    self.out[relu.id] = self.out[n.id]
            elif n.op == "relu":
                self.out[n.id] = self.out[n.inputs[0]]
            elif n.op in ("pool", "up"):
                self.out[n.id] = self._slab(n.c_out, self._ext(n.id))
        # gradient slabs ---------------------------------------------------
        self.gpre = {L.node.id: self._slab(L.cout, (L.D, L.H, L.W)) for L in self.layers if L.k == 3}
        self.gnode = {}
        for n in nodes:
            if n.op in ("pool", "concat"):
                self.gnode[n.id] = self._slab(n.c_out, self._ext(n.id))
        # head / loss -------------------------------------------------------
        head = self.by_id["head"]
        self.head = head
        self.head_in = head.node.inputs[0]
        hD, hH, hW = head.D, head.H, head.W
        self.nvox = self.B * hD * hH * hW
        # u8 class labels (the one-hot of training.py:68-69 is never materialised: the head
        # kernels compare the label, 1 B per voxel instead of 4*ncls) + a sticky error flag set
        # by the head forward when a label is >= ncls (np.eye(ncls)[labels] raises)
        self.labels = torch.zeros(self.nvox, dtype=torch.uint8, device=dev)
        self.label_err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.n_part = int(_lib.load().vm_head_partials_count(self.B, hD, hH, hW))
        self.partials = torch.zeros(self.n_part * (3 * self.ncls + 1), dtype=torch.float32, device=dev)
        self.stats = torch.zeros(3 * self.ncls + 1, dtype=torch.float32, device=dev)
        self.hw_width = head.cin * self.ncls + self.ncls
        self.hpartials = torch.zeros(self.n_part * self.hw_width, dtype=torch.float32, device=dev)
        self.hgrad = torch.zeros(self.hw_width, dtype=torch.float32, device=dev)
        self.repack()

    # ------------------------------------------------------------------ kernels
    def _st(self):
        return _lib.stream_ptr()

    def _k(self, kind, label, flops, nbytes, name, *args):
        """Launch ``name(*args, stream)``; in record mode, log it for per-kernel timing."""
        if self._rec is not None:
            self._rec.append((kind, label, flops, nbytes, name, args))
        _lib.call(name, *args, self._st())

    def _pack_table(self):
        """Device job table for vm_pack_weights_batch (one launch repacks every layer)."""
        if getattr(self, "_pack_jobs", None) is not None:
            return self._pack_jobs, self._pack_n, self._pack_total
        dt = np.dtype([("w", "<u8"), ("packed", "<u8"), ("cin", "<i4"), ("cout", "<i4"), ("flip", "<i4"),
                       ("pad", "<i4"), ("begin", "<i8")])
        rows, begin = [], 0
        for L in self.layers:
            if L.k != 3:
                continue
            for flip, buf in ((0, L.wp), (1, L.wpt)):
                ci, co = (L.cout, L.cin) if flip else (L.cin, L.cout)
                n = int(_lib.call_size("vm_packed_weights_bytes", ci, co)) // 2
                rows.append((L.w.data_ptr(), buf.data_ptr(), L.cin, L.cout, flip, 0, begin))
                begin += n
        arr = np.array(rows, dtype=dt)
        self._pack_jobs = torch.from_numpy(arr.view(np.uint8).copy()).to(self.device)
        self._pack_n, self._pack_total = len(rows), begin
        return self._pack_jobs, self._pack_n, self._pack_total

    def repack(self):
        """Refresh the derived conv operands from the fp32 master weights."""
        if self.conv_impl == "tc":
            jobs, n, total = self._pack_table()
            self._k("pack", "all", 0, 0, "vm_pack_weights_batch", _lib.ptr(jobs), n, total)
            return
        for L in self.layers:
            if L.k != 3:
                continue
            nb = 4 * L.nk
            if self.conv_impl == "tc":
                self._k("pack", L.node.id, 0, nb, "vm_pack_weights", _lib.ptr(L.w), _lib.ptr(L.wp), L.cin, L.cout, 0)
                self._k("pack", L.node.id, 0, nb, "vm_pack_weights", _lib.ptr(L.w), _lib.ptr(L.wpt), L.cin, L.cout, 1)
            else:
                self._k("pack", L.node.id, 0, nb, "vm_weight_flip_transpose", _lib.ptr(L.w), _lib.ptr(L.wt), 3,
                        L.cin, L.cout)

    def _conv_flops(self, L):
        return 2.0 * self.B * L.D * L.H * L.W * 27 * L.cin * L.cout

    def _fused_halo(self):
        """Peer-memory depth halo fused into the tensor-core convs (producer epilogue pushes,
        consumer waits): the transport and the conv path support it."""
        return (self.has_halo and self.fuse_halo and self.conv_impl == "tc"
                and isinstance(self.halo, PeerDepthHalo))

    def _exchanged_ptrs(self):
        """Slabs exchanged whole before a k=3 conv / dgrad reads them (fused-push candidates)."""
        if getattr(self, "_xptrs", None) is None:
            ptrs = set()
            for n in self.graph.nodes:
                if n.op == "conv" and n.k == 3:
                    ptrs.add(self.out[n.inputs[0]].ptr)
                    if n.inputs[0] != "input":
                        ptrs.add(self.gpre[n.id].ptr)
            self._xptrs = ptrs
        return self._xptrs

    def _conv(self, x, L, y, flags, mask=None, dgrad=False, planes=None, wait=None):
        cin, cout = (L.cout, L.cin) if dgrad else (L.cin, L.cout)
        mp = mask.p() if mask is not None else None
        mb = mask.bstride if mask is not None else 0
        kind = "conv_dgrad" if dgrad else "conv_fwd"
        nd = planes[1] if planes is not None else L.D
        vox = self.B * nd * L.H * L.W
        nbytes = 2.0 * vox * (cin + cout + (cout if mask is not None else 0))
        flops = self._conv_flops(L) * nd / L.D
        if planes is not None:  # output planes [d0, d0 + nd) (tensor-core path)
            w = L.wpt if dgrad else L.wp
            self._k(kind, L.node.id, flops, nbytes, "vm_conv3d_fwd_tc_range", x.p(), x.bstride, _lib.ptr(w),
                    _lib.ptr(L.b), y.p(), y.bstride, mp, mb, self.B, cin, cout, L.D, L.H, L.W, planes[0], nd, flags,
                    _lib.ptr(self.conv_ws), self.conv_ws_bytes)
        elif self.conv_impl == "tc" and L.c1 and not dgrad:
            self._k(kind, L.node.id, self._conv_flops(L), nbytes, "vm_conv3d_fwd_c1", _lib.ptr(self.x1), 0,
                    _lib.ptr(L.w), _lib.ptr(L.b), y.p(), y.bstride, self.B, cout, L.D, L.H, L.W, flags)
        elif self.conv_impl == "tc":
            w = L.wpt if dgrad else L.wp
            push = None
            if self._fused_halo() and y.ptr in self._exchanged_ptrs():
                push = self.halo.reserve_push(y)  # this conv pushes y's boundary layers itself
            link = HaloLinkC.of(push, wait)
            if link is not None:
                if getattr(self, "_links", None) is None:
                    self._links = {}
                self._links[(L.index, dgrad)] = link  # alive for recorded re-launches (profile_kernels)
                self._k(kind, L.node.id, self._conv_flops(L), nbytes, "vm_conv3d_fwd_tc_link", x.p(), x.bstride,
                        _lib.ptr(w), _lib.ptr(L.b), y.p(), y.bstride, mp, mb, self.B, cin, cout, L.D, L.H, L.W,
                        flags, _lib.ptr(self.conv_ws), self.conv_ws_bytes, ctypes.addressof(link))
            else:
                self._k(kind, L.node.id, self._conv_flops(L), nbytes, "vm_conv3d_fwd_tc_ws", x.p(), x.bstride,
                        _lib.ptr(w), _lib.ptr(L.b), y.p(), y.bstride, mp, mb, self.B, cin, cout, L.D, L.H, L.W,
                        flags, _lib.ptr(self.conv_ws), self.conv_ws_bytes)
        else:
            w = L.wt if dgrad else L.w
            self._k(kind, L.node.id, self._conv_flops(L), nbytes, "vm_conv3d_fwd_simt", self.dt, x.p(), x.bstride,
                    _lib.ptr(w), _lib.ptr(L.b), y.p(), y.bstride, mp, mb, self.B, cin, cout, L.D, L.H, L.W, flags)

    def _wgrad(self, x, L, g):
        vox = self.B * L.D * L.H * L.W
        nbytes = 2.0 * vox * (L.cin + L.cout) + 4.0 * (L.nk + L.cout)
        if self.conv_impl == "tc" and L.c1:
            f = getattr(self, "_fin", None)
            if f is not None and f["done"][0] is not None:  # a deferred finalize may still read wgrad_ws
                torch.cuda.current_stream().wait_event(f["done"][0])
            self._k("conv_wgrad", L.node.id, self._conv_flops(L), nbytes, "vm_conv3d_wgrad_c1", _lib.ptr(self.x1),
                    0, g.p(), g.bstride, _lib.ptr(L.gw), _lib.ptr(L.gb), _lib.ptr(self.wgrad_ws), self.B, L.cout, L.D,
                    L.H, L.W)
        elif self.conv_impl == "tc" and getattr(self, "_fin", None) is not None:
            # main kernel on this (side) stream into workspace i % 2; its finalize on the finalize
            # stream, so the next layer's weight gradient does not wait for it
            f = self._fin
            i = f["n"]
            f["n"] += 1
            ws = self.wgrad_ws if i % 2 == 0 else self.wgrad_ws2
            side = torch.cuda.current_stream()
            if f["done"][i % 2] is not None:  # the finalize that last read this workspace
                side.wait_event(f["done"][i % 2])
            self._k("conv_wgrad", L.node.id, self._conv_flops(L), nbytes, "vm_conv3d_wgrad_tc_phase", x.p(),
                    x.bstride, g.p(), g.bstride, _lib.ptr(L.gw), _lib.ptr(L.gb), _lib.ptr(ws), self.B, L.cin,
                    L.cout, L.D, L.H, L.W, 1)
            ev = torch.cuda.Event()
            ev.record(side)
            fs = self._fin_stream()
            fs.wait_event(ev)
            with torch.cuda.stream(fs):
                self._k("conv_wgrad", L.node.id, 0, 0, "vm_conv3d_wgrad_tc_phase", x.p(), x.bstride, g.p(),
                        g.bstride, _lib.ptr(L.gw), _lib.ptr(L.gb), _lib.ptr(ws), self.B, L.cin, L.cout, L.D, L.H,
                        L.W, 2)
                done = torch.cuda.Event()
                done.record(fs)
            f["done"][i % 2] = done
            f["last"] = done
        elif self.conv_impl == "tc":
            self._k("conv_wgrad", L.node.id, self._conv_flops(L), nbytes, "vm_conv3d_wgrad_tc", x.p(), x.bstride,
                    g.p(), g.bstride, _lib.ptr(L.gw), _lib.ptr(L.gb), _lib.ptr(self.wgrad_ws), self.B, L.cin,
                    L.cout, L.D, L.H, L.W)
        else:
            self._k("conv_wgrad", L.node.id, self._conv_flops(L), nbytes, "vm_conv3d_wgrad_simt", self.dt, x.p(),
                    x.bstride, g.p(), g.bstride, _lib.ptr(L.gw), _lib.ptr(L.gb), _lib.ptr(self.wgrad_ws), self.B,
                    L.cin, L.cout, L.D, L.H, L.W)

    def _halo(self, s, tag):
        if self.has_halo:
            self.halo.forward(s, tag)

    def halo_bytes_per_step(self, forward_only=False):
        """Bytes this rank sends per step (3-phase protocol, fwd + bwd, slab channel padding included)."""
        if not self.has_halo:
            return 0
        total = 0
        for n in self.graph.nodes:
            if n.op != "conv" or n.k != 3:
                continue
            L = self.by_id[n.id]
            cur = [L.D, L.H, L.W]
            cg = (L.cin + 7) // 8
            per = 0
            for i in range(3):
                lo, hi = self.nbrs.get(1 + i, (None, None))
                area = 1
                for j in range(3):
                    if j != i:
                        area *= cur[j]
                per += area * ((lo is not None) + (hi is not None))
                cur[i] += 2
            nbytes = per * cg * 8 * self.B * torch.tensor([], dtype=self.dtype).element_size()
            total += nbytes * (1 if (n.inputs[0] == "input" or forward_only) else 2)
        return total

    def _zero_margins(self, s):
        if self.has_halo:
            self.halo.zero(s)

    @staticmethod
    def _nbr26(ctx, layout, nbr6):
        """Face, edge and corner neighbour ranks (vm_halo_slab_fwd26 order) of this rank: the
        mesh coordinate moved by s along the mesh axes of the split spatial dims."""
        if ctx is None or layout is None:
            return None
        axes = [layout.axis_for(d) for d in ("x", "y", "z")]
        mesh = ctx.mesh

        def rank_at(s):
            coord = list(ctx.coord)
            for i, si in enumerate(s):
                if si:
                    j = mesh.axis_index[axes[i]]
                    coord[j] += si
            return mesh.rank_of[tuple(coord)]

        return nbr26_of(nbr6, rank_at)

    def use_nccl(self, comm, nbr6=None, ar_comm=None):
        """Route the halo and the collectives through NCCL communicator ``comm`` (an
        ncclComm_t).  ``nbr6`` overrides the neighbour ranks: a 1-rank communicator with the
        rank as its own lo and hi neighbour gives periodic halos on one GPU (the single-GPU
        emulation of a split: same pack / NCCL / unpack work, no NVLink wire time)."""
        if nbr6 is not None:
            self.halo = SlabHalo(nbr6, ctx=self.ctx, comm=comm, nbr26=nbr26_of(nbr6))
            for i in range(3):
                lo, hi = nbr6[2 * i], nbr6[2 * i + 1]
                if lo >= 0 or hi >= 0:
                    self.nbrs[1 + i] = (lo if lo >= 0 else None, hi if hi >= 0 else None)
            self.has_halo = self.halo.active
            if self.has_halo:  # a halo'd first conv reads the 8-channel input slab (margins exchanged)
                for L in self.layers:
                    L.c1 = False
                self.input_slab_needed = True
        else:
            self.halo.comm = comm
        self.comm = comm
        self.ar_comm = ar_comm
        self._reserve_halo()

    def use_peer_halo(self, nbr6=None, group=None):
        """Depth-split halos through peer memory (halo.PeerDepthHalo, vm_halo_depth_push)
        instead of NCCL.  ``nbr6`` given: a single-GPU emulation whose neighbours are this rank
        itself (periodic halos, same launches and bytes); otherwise the mesh's own neighbours,
        mapped over CUDA IPC (spmd, one process per GPU)."""
        emulate = nbr6 is not None
        if not emulate:
            peer = PeerDepthHalo(self.halo.nbr6, self.device, self_peers=False)
            if peer.active:
                peer.connect(self._halo_slabs(), group)  # collective: every rank calls it
        else:
            peer = PeerDepthHalo(nbr6, self.device, self_peers=True)
            for i in range(3):
                lo, hi = nbr6[2 * i], nbr6[2 * i + 1]
                if lo >= 0 or hi >= 0:
                    self.nbrs[1 + i] = (lo if lo >= 0 else None, hi if hi >= 0 else None)
        self.halo = peer
        self.has_halo = peer.active
        if self.has_halo:  # a halo'd first conv reads the 8-channel input slab (margins exchanged)
            for L in self.layers:
                L.c1 = False
            self.input_slab_needed = True

    def _halo_slabs(self):
        slabs = [self.out[n.inputs[0]] for n in self.graph.nodes if n.op == "conv" and n.k == 3]
        return slabs + list(self.gpre.values())

    def _reserve_halo(self):
        if self.halo.comm is None:
            return
        self.halo.reserve(self._halo_slabs())

    def _split_planes(self, D):
        """Interior / boundary split of a conv's output planes around a depth-only halo."""
        n = self.halo.nbr6
        depth_only = (n[0] >= 0 or n[1] >= 0) and max(n[2:]) < 0
        return (self.overlap_halo and self.has_halo and depth_only and self.conv_impl == "tc"
                and D >= self.overlap_min_planes and not isinstance(self.halo, PeerDepthHalo))

    def graph_capturable(self):
        return self.ctx is None or self.ctx.mesh.worker_count == 1 or self.comm is not None

    def _sm_budget(self):
        if getattr(self, "_nsm", None) is None:
            self._nsm = int(_lib.load().vm_num_sms(self.device.index or 0))
        return max(1, self._nsm - self.halo_sm_reserve)

    def _comm_stream(self):
        if getattr(self, "_cstream", None) is None:
            self._cstream = torch.cuda.Stream(device=self.device)
        return self._cstream

    def _ar_stream(self):
        if getattr(self, "_arstream", None) is None:
            self._arstream = torch.cuda.Stream(device=self.device)
        return self._arstream

    def _halo_conv(self, x, L, y, flags, mask=None, dgrad=False, tag="halo"):
        """Halo of ``x`` then conv(x): with a depth-only split the exchange runs on the comm
        stream while the interior output planes compute, then the two boundary planes."""
        if self._fused_halo() and not (L.c1 and not dgrad):
            # the producer of x pushed its boundary layers (the conv waits for the
            # neighbours' pushes), or a standalone push runs here
            wait = self.halo.consume(x)
            self._conv(x, L, y, flags, mask=mask, dgrad=dgrad, wait=wait)
            return
        if not self._split_planes(L.D) or (L.c1 and not dgrad):
            self._halo(x, tag)
            self._conv(x, L, y, flags, mask=mask, dgrad=dgrad)
            return
        main = torch.cuda.current_stream()
        comm = self._comm_stream()
        ready = torch.cuda.Event()
        ready.record(main)
        lib = _lib.load()
        prev = lib.vm_set_conv_sm_limit(self._sm_budget())  # leave SMs to the exchange kernels
        try:
            self._conv(x, L, y, flags, mask=mask, dgrad=dgrad, planes=(1, L.D - 2))
        finally:
            lib.vm_set_conv_sm_limit(prev)
        comm.wait_event(ready)
        with torch.cuda.stream(comm):
            self._halo(x, tag)
            done = torch.cuda.Event()
            done.record(comm)
        main.wait_event(done)
        self._conv(x, L, y, flags, mask=mask, dgrad=dgrad, planes=(0, 1))
        self._conv(x, L, y, flags, mask=mask, dgrad=dgrad, planes=(L.D - 1, 1))

    # ------------------------------------------------------------------ inputs
    def load_inputs(self, image, labels):
        """image: device f32 [B,D,H,W,Cin] (local block); labels: device u8 [B,D,H,W] class
        indices, or a one-hot f32 [B,D,H,W,ncls] (test convenience: its argmax is taken)."""
        x = self.x_in
        self._check_shape(image, labels)
        if self.input_slab_needed:
            self._k("io", "image", 0, 0, "vm_dense_to_slab", _lib.ptr(image.contiguous()), _lib.VM_F32, x.p(),
                    self.dt, x.bstride, self.B, x.C, x.D, x.H, x.W, 1)
        self._compact_input(image.contiguous())
        if labels.dtype != torch.uint8:
            labels = labels.argmax(dim=-1).to(torch.uint8)
        self.labels.copy_(labels.reshape(-1))

    def _check_shape(self, image, labels):
        x = self.x_in
        want = (self.B, x.D, x.H, x.W)
        if tuple(image.shape[:4]) != want or tuple(labels.shape[:4]) != want:
            raise VoxmeshError(f"input block {tuple(image.shape)} / labels {tuple(labels.shape)} do not match the "
                               f"step's local block {want} (batch, D, H, W)")

    def _compact_input(self, image):
        if self.x1 is not None:
            x = self.x_in
            self._k("io", "image", 0, 0, "vm_dense_to_compact1", _lib.ptr(image), _lib.ptr(self.x1), self.B, x.D,
                    x.H, x.W)

    def upload(self, image_host, labels_host):
        """Public-API input path: host f32 image [B,D,H,W,Cin] + u8 labels [B,D,H,W]
        -> (pinned) H2D -> slab + on-device one-hot (training.py:68-69, :276-279)."""
        self._stage_h2d(image_host, labels_host)
        self._consume_staged()

    # Double-buffered host->device staging: the H2D of step k+1's inputs runs on a copy
    # stream while step k computes (a data loader's prefetch); each step still moves its own
    # input bytes and reads its loss back.
    def _stage_bufs(self, image_host, labels_host):
        self._check_shape(image_host, labels_host)
        if getattr(self, "_stage", None) is None:
            self._stage = [(torch.empty(tuple(image_host.shape), dtype=torch.float32, device=self.device),
                            torch.empty(tuple(labels_host.shape), dtype=torch.uint8, device=self.device))
                           for _ in range(2)]
            self._copy_stream = torch.cuda.Stream(device=self.device)
            self._copied = [None, None]   # event: H2D into buffer i done
            self._consumed = [None, None]  # event: buffer i read by the compute stream
            self._next = 0                 # buffer the next step consumes
            self._pending = None           # buffer holding a prefetched input, if any

    def _stage_h2d(self, image_host, labels_host, on_copy_stream=False):
        self._stage_bufs(image_host, labels_host)
        i = self._next if self._pending is None else 1 - self._pending
        img, lab = self._stage[i]
        if on_copy_stream:
            cs = self._copy_stream
            if self._consumed[i] is not None:
                cs.wait_event(self._consumed[i])
            with torch.cuda.stream(cs):
                img.copy_(image_host, non_blocking=True)
                lab.copy_(labels_host, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
            self._copied[i] = ev
        else:
            img.copy_(image_host, non_blocking=True)
            lab.copy_(labels_host, non_blocking=True)
            self._copied[i] = None
        self._pending = i

    def _consume_staged(self):
        i = self._pending
        img, lab = self._stage[i]
        if self._copied[i] is not None:
            torch.cuda.current_stream().wait_event(self._copied[i])
        x = self.x_in
        if self.input_slab_needed:
            self._k("io", "image", 0, 0, "vm_dense_to_slab", _lib.ptr(img), _lib.VM_F32, x.p(), self.dt,
                    x.bstride, self.B, x.C, x.D, x.H, x.W, 1)
        self._compact_input(img)
        self.labels.copy_(lab.reshape(-1), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._consumed[i] = ev
        self._pending = None
        self._next = 1 - i

    def train_step_host(self, image_host, labels_host, replay=None, next_inputs=None):
        """One step through the public API: H2D inputs, step (or graph replay), D2H loss.

        ``next_inputs = (image_host, labels_host)`` of the following step starts that step's
        H2D on a copy stream while this step computes; the following call then consumes the
        prefetched buffer (its own ``image_host``/``labels_host`` must be those tensors)."""
        if self._has_prefetch(image_host):
            self._consume_staged()
        else:
            self.upload(image_host, labels_host)
        if replay is not None:
            replay()
        else:
            self.step()
        if next_inputs is not None:
            self._stage_h2d(next_inputs[0], next_inputs[1], on_copy_stream=True)
            self._prefetched_src = next_inputs[0]
        return self.loss()[0]

    def train_loop_host(self, batches, replay=None):
        """Pipelined public-API training loop over host batches ``[(image, labels), ...]``
        (pinned): every step moves its inputs host->device (step k+1's on a copy stream while
        step k computes) and its loss statistics device->host (async copy into pinned memory);
        the host reads step k's loss while step k+1 runs, like a training loop that logs one
        step behind.  Returns the per-step (combined, dice, ce) losses."""
        batches = list(batches)
        if getattr(self, "_loss_host", None) is None:
            self._loss_host = [torch.empty(self.stats.numel(), dtype=self.stats.dtype).pin_memory()
                               for _ in range(2)]
            self._err_host = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(2)]
        out, prev = [], None
        self.upload(*batches[0])
        for k in range(len(batches)):
            if k > 0:
                self._consume_staged()
            if replay is not None:
                replay()
            else:
                self.step()
            buf, err = self._loss_host[k % 2], self._err_host[k % 2]
            buf.copy_(self.stats, non_blocking=True)
            err.copy_(self.label_err, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            if k + 1 < len(batches):
                self._stage_h2d(*batches[k + 1], on_copy_stream=True)
            if prev is not None:
                prev[0].synchronize()
                self._check_labels(int(prev[2][0]))
                out.append(self._loss_from(prev[1].numpy()))
            prev = (ev, buf, err)
        prev[0].synchronize()
        self._check_labels(int(prev[2][0]))
        out.append(self._loss_from(prev[1].numpy()))
        return out

    # ------------------------------------------------------------------ public training loop
    # training.train_loop drives these: the host batch goes into persistent pinned buffers
    # (two slots), its H2D + slab kernels run on this rank's stream, the step replays a captured
    # CUDA graph when the transport allows it (one rank, or NCCL through the C ABI), and the
    # loss statistics come back by an async D2H that the caller collects one step later.
    def capture(self):
        """Capture step() as a CUDA graph (None when the transport cannot be captured: the
        threads mesh exchanges through host queues).  Replays run on the current stream."""
        if self.ctx is not None and self.ctx.mesh.worker_count > 1 and not self.graph_capturable():
            return None
        import gc

        # a CUDAGraph freed by the garbage collector in the middle of the capture (another
        # step's graph) would invalidate it: collect first; thread-local capture mode so that
        # other threads' CUDA calls (the threads mesh captures one rank per thread) are legal
        gc.collect()
        cur = torch.cuda.current_stream(self.device)
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                self.step()
        cur.wait_stream(s)
        return g

    def launch_host_step(self, image_np, labels_np, replay=None):
        """Stage numpy host blocks -> pinned -> device, run one step, start the D2H of its
        loss statistics; returns a handle for ``collect`` (no host sync)."""
        if getattr(self, "_loop", None) is None:
            self._loop = {"slot": 0, "pinned": [None, None], "ev": [None, None],
                          "stats": [torch.empty(self.stats.numel(), dtype=torch.float32).pin_memory() for _ in range(2)],
                          "err": [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(2)],
                          "skip": [torch.zeros(len(self.layers), dtype=torch.int32).pin_memory() for _ in range(2)]}
        lp = self._loop
        i = lp["slot"]
        lp["slot"] = 1 - i
        if lp["ev"][i] is not None:
            lp["ev"][i].synchronize()  # the step that last used slot i has finished (H2D + D2H)
        if lp["pinned"][i] is None or tuple(lp["pinned"][i][0].shape) != tuple(image_np.shape):
            lp["pinned"][i] = (torch.empty(tuple(image_np.shape), dtype=torch.float32).pin_memory(),
                               torch.empty(tuple(labels_np.shape), dtype=torch.uint8).pin_memory())
        img, lab = lp["pinned"][i]
        np.copyto(img.numpy(), image_np, casting="same_kind")
        np.copyto(lab.numpy(), labels_np, casting="unsafe")
        self.upload(img, lab)
        if replay is not None:
            replay()
        else:
            self.step()
        lp["stats"][i].copy_(self.stats, non_blocking=True)
        lp["err"][i].copy_(self.label_err, non_blocking=True)
        lp["skip"][i].copy_(self.skip_flags, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        lp["ev"][i] = ev
        return i, ev

    def collect(self, handle):
        """(combined, dice, ce), skipped layer ids of a launched step (waits for it)."""
        i, ev = handle
        lp = self._loop
        ev.synchronize()
        self._check_labels(int(lp["err"][i][0]))
        flags = lp["skip"][i].numpy()
        return self._loss_from(lp["stats"][i].numpy()), [L.node.id for L, f in zip(self.layers, flags) if f]

    def _has_prefetch(self, image_host):
        return (getattr(self, "_pending", None) is not None and self._copied[self._pending] is not None
                and getattr(self, "_prefetched_src", None) is image_host)

    # ------------------------------------------------------------------ passes
    def forward(self):
        prev = _lib.load().vm_set_pdl(int(self.pdl_forward))
        try:
            self._forward_nodes()
        finally:
            _lib.load().vm_set_pdl(prev)

    def _forward_nodes(self):
        if self.has_halo and hasattr(self.halo, "begin_step"):
            self.halo.begin_step()
        for n in self.graph.nodes:
            if n.op == "conv" and n.k == 3:
                x = self.out[n.inputs[0]]
                self._halo_conv(x, self.by_id[n.id], self.out[n.id], _lib.VM_CONV_RELU)
            elif n.op == "pool":
                x, y = self.out[n.inputs[0]], self.out[n.id]
                nb = 2.0 * self.B * x.D * x.H * x.W * x.C * 9 / 8
                self._k("pool_fwd", n.id, 0, nb, "vm_maxpool2_fwd", self.dt, x.p(), x.bstride, y.p(), y.bstride,
                        self.B, x.C, x.D, x.H, x.W)
            elif n.op == "up":
                x, y = self.out[n.inputs[0]], self.out[n.id]
                nb = 2.0 * self.B * x.D * x.H * x.W * x.C * 9
                self._k("up_fwd", n.id, 0, nb, "vm_upsample2_fwd", self.dt, x.p(), x.bstride, y.p(), y.bstride,
                        self.B, x.C, x.D, x.H, x.W)
            elif n.op == "concat":
                c_up, aligned = self.cat_parts[n.id]
                if not aligned:
                    self._concat_copy(n)
        h = self.head
        y = self.out[self.head_in]
        probs = None
        if self.keep_probs:
            if getattr(self, "probs", None) is None:
                self.probs = torch.empty(self.nvox * self.ncls, dtype=torch.float32, device=self.device)
            probs = _lib.ptr(self.probs)
        if self.keep_pred and self.pred is None:
            self.pred = torch.empty(self.nvox, dtype=torch.uint8, device=self.device)
        nb = 2.0 * self.nvox * h.cin + 1.0 * self.nvox
        self._k("head_fwd", "head", 2.0 * self.nvox * h.cin * self.ncls, nb, "vm_head_fwd", self.dt, y.p(), y.bstride,
                _lib.ptr(h.w), _lib.ptr(h.b), _lib.ptr(self.labels), _lib.ptr(self.label_err), probs,
                _lib.ptr(self.pred) if self.keep_pred else None, _lib.ptr(self.partials), self.B, h.cin,
                self.ncls, h.D, h.H, h.W, self.clamp)
        self._k("reduce", "stats", 0, 0, "vm_reduce_rows", _lib.ptr(self.partials), self.n_part, 3 * self.ncls + 1,
                _lib.ptr(self.stats))
        if self.comm is not None and self.stats_axes is None:  # training.py:337 over NCCL
            self._k("coll", "stats", 0, 0, "vm_allreduce_f32", ctypes.c_void_p(self.comm), _lib.ptr(self.stats),
                    self.stats.numel())
        elif self.ctx is not None and self.ctx.mesh.worker_count > 1 and self.stats_axes != ():
            red = self.ctx.all_reduce_sum(self.stats, axes=self.stats_axes, tag="loss-stats")
            if red is not self.stats:
                self.stats.copy_(red)

    def backward(self, dprobs=None):
        """Backward of the step's loss; ``dprobs`` (device f32 [B,D,H,W,ncls]) replaces the
        loss gradient with a given dL/dprobs (the worker-level API, unet.run_backward_local)."""
        prev = _lib.load().vm_set_pdl(int(self.pdl_backward))
        try:
            self._backward_nodes(dprobs)
        finally:
            _lib.load().vm_set_pdl(prev)

    def _backward_nodes(self, dprobs=None):
        h = self.head
        y = self.out[self.head_in]
        last = self.graph.node(self.head_in)
        last_conv = last.inputs[0] if last.op == "relu" else last.id
        g = self.gpre[last_conv]
        nb = 4.0 * self.nvox * h.cin + 1.0 * self.nvox
        if dprobs is not None:
            dp = dprobs.contiguous().float()
            self._k("head_bwd", "head", 4.0 * self.nvox * h.cin * self.ncls, nb, "vm_head_bwd_dprobs", self.dt, y.p(),
                    y.bstride, _lib.ptr(h.w), _lib.ptr(h.b), _lib.ptr(dp), g.p(), g.bstride, _lib.ptr(self.hpartials),
                    self.B, h.cin, self.ncls, h.D, h.H, h.W, 1)
        else:
            self._k("head_bwd", "head", 4.0 * self.nvox * h.cin * self.ncls, nb, "vm_head_bwd", self.dt, y.p(),
                    y.bstride, _lib.ptr(h.w), _lib.ptr(h.b), _lib.ptr(self.labels), _lib.ptr(self.stats), g.p(),
                    g.bstride, _lib.ptr(self.hpartials), self.B, h.cin, self.ncls, h.D, h.H, h.W, self.w_dice,
                    self.w_ce, self.total_voxels, self.dice_mask, self.clamp, 1)
        self._k("reduce", "head", 0, 0, "vm_reduce_rows", _lib.ptr(self.hpartials), self.n_part, self.hw_width,
                _lib.ptr(self.hgrad))
        # head grads: [C*ncls] kernel (DHWIO with k=1) then [ncls] bias — contiguous in the flat buffer
        h.gw.copy_(self.hgrad[: h.nk])
        h.gb.copy_(self.hgrad[h.nk :])
        # wgrad(x, g) and dgrad(g) of a conv are independent: the weight gradients run on a
        # side stream (joined before SGD), which fills the SMs the small deep-level kernels
        # leave idle.  Without a halo, wgrad starts with the layer's dgrad.  With a halo, the
        # exchange writes g's margins and wgrad reads them as zeros: halo -> dgrad -> zero the
        # margins on the main stream, then wgrad on the side stream behind a per-layer event,
        # so the main stream never waits for a weight gradient.  Over NCCL the weight
        # gradients are all-reduced in buckets on their own stream and communicator as soon
        # as a bucket's last wgrad is done (unet.py:434-441), overlapping the rest of backward.
        main = torch.cuda.current_stream()
        side = self._side_stream() if self.overlap_wgrad else None
        buckets = self._grad_buckets() if (self.ar_comm is not None and side is not None) else {}
        self._fin = ({"n": 0, "done": [None, None], "last": None}
                     if (side is not None and self.defer_finalize and self.conv_impl == "tc") else None)
        if buckets:
            ar = self._ar_stream()
        # a transport whose margins the weight gradient never reads (peer-memory depth halo):
        # wgrad runs on the side stream while the main stream exchanges gy and runs dgrad
        concurrent = self.has_halo and getattr(self.halo, "wgrad_safe", False) and self.conv_impl == "tc"
        serial_halo = self.has_halo and not concurrent
        for n in reversed(self.graph.nodes):
            if n.op == "conv" and n.k == 3:
                L = self.by_id[n.id]
                x = self.out[n.inputs[0]]
                gp = self.gpre[n.id]
                src = n.inputs[0]
                if src != "input" and serial_halo:
                    self._dgrad(gp, L, src)
                    self._zero_margins(gp)
                    if side is not None:
                        ev = torch.cuda.Event()
                        ev.record(main)
                        side.wait_event(ev)
                if side is not None:
                    if not serial_halo:
                        side.wait_stream(main)
                    with torch.cuda.stream(side):
                        self._wgrad(x, L, gp)
                        if L.index in buckets:
                            ev = torch.cuda.Event()
                            ev.record(side)
                            ar.wait_event(ev)
                            if self._fin is not None and self._fin["last"] is not None:
                                ar.wait_event(self._fin["last"])  # the bucket's last finalize
                            lo, hi = buckets[L.index]
                            with torch.cuda.stream(ar):
                                self._k("coll", "grads", 0, 0, "vm_allreduce_f32", ctypes.c_void_p(self.ar_comm),
                                        _lib.ptr(self.grads[lo:hi]), hi - lo)
                else:
                    self._wgrad(x, L, gp)
                if src != "input" and not serial_halo:
                    self._dgrad(gp, L, src)
            elif n.op == "up":
                cat = next(c for c in self.consumers[n.id] if c.op == "concat")
                gcat = self.gnode[cat.id]
                c_up, aligned = self.cat_parts[cat.id]
                gup = self._window(gcat, 0, c_up, aligned, copy_from=cat.id, part="up")
                src = n.inputs[0]
                sn = self.graph.node(src)
                x = self.out[src]
                dst = self.gpre[sn.inputs[0]]
                nb = 2.0 * self.B * x.D * x.H * x.W * x.C * 10
                self._k("up_bwd", n.id, 0, nb, "vm_upsample2_bwd", self.dt, gup.p(), gup.bstride, x.p(), x.bstride,
                        dst.p(), dst.bstride, self.B, x.C, x.D, x.H, x.W)
            elif n.op == "pool":
                src = n.inputs[0]
                sn = self.graph.node(src)
                x = self.out[src]
                dst = self.gpre[sn.inputs[0]]
                gpool = self.gnode[n.id]
                cat = next((c for c in self.consumers[src] if c.op == "concat"), None)
                add = None
                if cat is not None:
                    c_up, aligned = self.cat_parts[cat.id]
                    add = self._window(self.gnode[cat.id], c_up, cat.c_out - c_up, aligned, copy_from=cat.id,
                                       part="skip")
                vin = self.B * x.D * x.H * x.W * x.C
                nb = 2.0 * vin * (1 + (1 if add else 0) + 1) + 2.0 * vin / 8
                self._k("pool_bwd", n.id, 0, nb, "vm_maxpool2_bwd", self.dt, x.p(), x.bstride, gpool.p(),
                        gpool.bstride, add.p() if add else None, add.bstride if add else 0, dst.p(), dst.bstride,
                        self.B, x.C, x.D, x.H, x.W, 1)

        if side is not None:
            main.wait_stream(side)
        if self._fin is not None:
            # join through the recorded events only: an unused finalize stream is not part of a
            # graph capture, and waiting on it would invalidate the capture
            for ev in self._fin["done"]:
                if ev is not None:
                    main.wait_event(ev)
            self._fin = None
        if buckets:
            main.wait_stream(ar)
        self._grads_reduced = bool(buckets)

    def _dgrad(self, gp, L, src):
        """Halo of the output gradient, then the data gradient (ops.py:100-114) with the
        producer's ReLU mask fused (ops.py:186-187)."""
        sn = self.graph.node(src)
        if sn.op == "relu":
            self._halo_conv(gp, L, self.gpre[sn.inputs[0]], _lib.VM_CONV_MASK | _lib.VM_CONV_NOBIAS,
                            mask=self.out[src], dgrad=True, tag="halo-bwd")
        else:  # pool or concat output gradient, unmasked
            self._halo_conv(gp, L, self.gnode[src], _lib.VM_CONV_NOBIAS, dgrad=True, tag="halo-bwd")

    def _grad_buckets(self):
        """{layer index closing a bucket: (flat lo, flat hi)}: contiguous runs of layers in
        backward order of >= bucket_bytes of fp32 gradients."""
        if getattr(self, "_buckets", None) is None:
            out, hi, size = {}, None, 0
            for L in reversed(self.layers):
                a, b = self.offsets_host[L.index], self.offsets_host[L.index + 1]
                hi = b if hi is None else hi
                size += 4 * (b - a)
                if size >= self.bucket_bytes or L.index == 0:
                    out[L.index] = (a, hi)
                    hi, size = None, 0
            self._buckets = out
        return self._buckets

    def _fin_stream(self):
        if getattr(self, "_fstream", None) is None:
            self._fstream = torch.cuda.Stream(device=self.device)
        return self._fstream

    def _side_stream(self):
        if getattr(self, "_wg_stream", None) is None:
            self._wg_stream = torch.cuda.Stream(device=self.device)
        return self._wg_stream

    def all_reduce_grads(self):
        """Sum the weight gradients over every mesh axis (unet.py:434-441); a no-op when the
        backward already all-reduced them in buckets."""
        if getattr(self, "_grads_reduced", False):
            return
        if self.comm is not None:
            self._k("coll", "grads", 0, 0, "vm_allreduce_f32", ctypes.c_void_p(self.comm), _lib.ptr(self.grads),
                    self.grads.numel())
        elif self.ctx is not None and self.ctx.mesh.worker_count > 1:
            red = self.ctx.all_reduce_sum(self.grads, tag="grads")
            if red is not self.grads:
                self.grads.copy_(red)

    def sgd(self):
        n = self.params.numel()
        self._k("sgd", "all", 0, 20.0 * n, "vm_sgd_momentum", _lib.ptr(self.params), _lib.ptr(self.moments),
                _lib.ptr(self.grads), _lib.ptr(self.offsets), len(self.layers), self.max_layer,
                _lib.ptr(self.skip_flags), self.lr, self.mu)
        self.repack()

    def step(self):
        """One train step on the resident inputs (fwd -> stats -> bwd -> grads -> SGD)."""
        self.forward()
        self.backward()
        self.all_reduce_grads()
        self.sgd()

    def profile_kernels(self, reps=5):
        """Per-launch device time of every kernel of one step: each launch is captured
        alone in a CUDA graph and replayed ``reps`` times between CUDA events."""
        self._rec = []
        try:
            self.step()
        finally:
            rec, self._rec = self._rec, None
        torch.cuda.synchronize()
        rows = []
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for kind, label, flops, nbytes, name, args in rec:
                if kind == "coll":  # a collective replayed on one rank alone would wait for its peers
                    continue
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(reps):
                        _lib.call(name, *args, self._st())
                g.replay()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                g.replay()
                e1.record(s)
                e1.synchronize()
                rows.append({"kind": kind, "layer": label, "ms": e0.elapsed_time(e1) / reps, "flops": flops,
                             "bytes": nbytes})
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        return rows

    # ------------------------------------------------------------------ helpers
    def _window(self, s, c0, nc, aligned, copy_from=None, part=None):
        if aligned:
            return Slab(self.B, nc, s.D, s.H, s.W, self.dtype, self.device, parent=s, cg0=c0 // 8)
        key = (copy_from, part)
        if not hasattr(self, "_tmp"):
            self._tmp = {}
        if key not in self._tmp:
            self._tmp[key] = self._slab(nc, (s.D, s.H, s.W))
        t = self._tmp[key]
        self._copy_channels(s, c0, t, 0, nc)
        return t

    def _copy_channels(self, src, c0, dst, d0, nc):
        dense = src.interior()[..., c0 : c0 + nc].contiguous()
        if dst.C != nc or d0 != 0:
            full = dst.interior()
            full[..., d0 : d0 + nc] = dense
            dense = full
        _lib.call("vm_dense_to_slab", _lib.ptr(dense), _lib.VM_F32, dst.p(), self.dt, dst.bstride, self.B,
                  dst.C, dst.D, dst.H, dst.W, 1, self._st())

    def _concat_copy(self, n):
        up_id, skip_id = n.inputs
        cat = self.out[n.id]
        up, skip = self.out[up_id], self.out[skip_id]
        dense = torch.cat([up.interior(), skip.interior()], dim=-1).contiguous()
        _lib.call("vm_dense_to_slab", _lib.ptr(dense), _lib.VM_F32, cat.p(), self.dt, cat.bstride, self.B,
                  cat.C, cat.D, cat.H, cat.W, 1, self._st())

    # ------------------------------------------------------------------ readout
    def loss(self):
        """(combined, dice, ce) from the reduced statistics (training.py:95-107)."""
        self._check_labels(int(self.label_err.item()))
        return self._loss_from(self.stats.double().cpu().numpy())

    def _check_labels(self, flag):
        if flag:
            raise VoxmeshError(f"label volume holds a class index >= num_classes ({self.ncls}): "
                               "one_hot (training.py:68-69) would raise IndexError")

    def _loss_from(self, s):
        s = np.asarray(s, dtype=np.float64)
        c = self.ncls
        ks = [k for k in range(c) if (self.dice_mask >> k) & 1]
        ratios = [(2.0 * s[k] + 1e-6) / (s[c + k] + s[2 * c + k] + 1e-6) for k in ks]
        dice = 1.0 - sum(ratios) / len(ratios)
        ce = float(s[3 * c]) / self.total_voxels
        return self.w_dice * dice + self.w_ce * ce, dice, ce

    def param_dict(self):
        host = self.params.cpu().numpy()
        out = {}
        for L, a in zip(self.layers, self.offsets_host):
            out[L.node.id] = {
                "kernel": host[a : a + L.nk].reshape(L.k, L.k, L.k, L.cin, L.cout).copy(),
                "bias": host[a + L.nk : a + L.nk + L.cout].copy(),
            }
        return out

    def skipped_layers(self):
        """Conv ids whose gradients were non-finite in the last SGD step (training.py:202-219)."""
        flags = self.skip_flags.cpu().numpy()
        return [L.node.id for L, f in zip(self.layers, flags) if f]

    def moment_dict(self):
        """SGD momentum buffers in the reference layout {id: {"kernel", "bias"}}."""
        host = self.moments.cpu().numpy()
        return {
            L.node.id: {"kernel": host[a : a + L.nk].reshape(L.k, L.k, L.k, L.cin, L.cout).copy(),
                        "bias": host[a + L.nk : a + L.nk + L.cout].copy()}
            for L, a in zip(self.layers, self.offsets_host)
        }

    def load_state(self, params=None, moments=None):
        """Install reference-layout parameters and/or momentum buffers (checkpoint resume,
        ``training.install_params``); the conv operands are repacked."""
        for store, buf in ((params, self.params), (moments, self.moments)):
            if store is None:
                continue
            host = buf.cpu().numpy()
            for L, a in zip(self.layers, self.offsets_host):
                blob = store[L.node.id]
                host[a : a + L.nk] = np.asarray(blob["kernel"], dtype=np.float32).reshape(-1)
                host[a + L.nk : a + L.nk + L.cout] = np.asarray(blob["bias"], dtype=np.float32)
            buf.copy_(torch.from_numpy(host))
        if params is not None:
            self.repack()

    def grad_dict(self):
        host = self.grads.cpu().numpy()
        return {
            L.node.id: (host[a : a + L.nk].reshape(L.k, L.k, L.k, L.cin, L.cout).copy(),
                        host[a + L.nk : a + L.nk + L.cout].copy())
            for L, a in zip(self.layers, self.offsets_host)
        }
