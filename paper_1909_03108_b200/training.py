"""Training loop, checkpoints and evaluation around the GPU train step (SURVEY §8(f) rows 1
and 3: the caller of the hot path and the step after it).

Mirrors ``voxmesh.training`` (training.py) for a user switching over:

* ``TrainConfig`` / ``TrainState`` / ``LossWeights`` (training.py:43-50, :364-387);
* ``save_checkpoint`` / ``load_checkpoint`` write and read the reference's on-disk format,
  one directory per checkpoint with ``{param,moment}__{node}__{kernel,bias}.npy`` blobs and
  a ``manifest.json`` (training.py:414-439), so either implementation resumes from the
  other's checkpoints;
* ``BatchSource`` draws the same batches from (seed, step): per-epoch permutations seeded
  ``SeedSequence([seed, 7919, epoch])`` (training.py:241-279), which is what makes resume
  bitwise;
* ``train_loop`` (training.py:442-533) runs ``UNetStep`` on every rank of the graph's mesh
  (threads: one worker thread + CUDA stream per rank; spmd: this process's rank), streams
  ``metrics.csv`` and ``run.json`` in the reference's formats and checkpoints every
  ``checkpoint_every`` steps;
* ``evaluate`` (training.py:543-602) runs the forward pass on the GPU and reports hard
  tumour Dice per case and pooled (``hard_dice`` / ``dice_per_case`` / ``dice_global``,
  training.py:166-194) plus the mean loss.

The arithmetic is the GPU step's (bf16 storage, fp32 accumulation; ``compute_dtype="f32"``
selects the fp32 CUDA-core kernels).  ``TrainConfig.augment`` (a ``SynthConfig``) runs the
tumour remove / synthesise augmentation (``augment.py``, GPU kernels) on every sample with
the reference's per-sample seed ``SeedSequence([seed, 104729, global index])``
(training.py:266-273); its outputs are bitwise the reference's.
"""

from __future__ import annotations

import json
import os
import time
import warnings
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import HaloError, ShardingError, VoxmeshError

DICE_EPS = 1e-6


@dataclass(frozen=True)
class LossWeights:
    dice: float = 0.9
    ce: float = 0.1

    def __post_init__(self):
        if self.dice < 0 or self.ce < 0:
            raise VoxmeshError(f"loss weights must be non-negative: {self}")


@dataclass
class TrainConfig:
    """Same fields and defaults as the reference (training.py:364-379), plus
    ``compute_dtype`` ("bf16": tensor-core path, "f32": CUDA-core fp32 path)."""

    steps: int = 200
    batch_size: int = 1
    lr: float = 0.003
    momentum: float = 0.9
    seed: int = 0
    dice_classes: tuple = (1, 2)
    loss_weights: LossWeights = field(default_factory=LossWeights)
    prob_clamp: float = 1e-12
    dtype: str = "f32"
    augment: object = None
    checkpoint_every: int = 0
    log_every: int = 1
    out_dir: str = None
    phase_barrier: bool = True
    compute_dtype: str = "bf16"


@dataclass
class TrainState:
    step: int
    params: dict
    moments: dict
    history: list = field(default_factory=list)


# ---------------------------------------------------------------------------- losses
def one_hot(labels, num_classes, dtype=np.float32):
    """training.py:68-69."""
    return np.eye(num_classes, dtype=dtype)[labels]


def _dev(a):
    """(device f32 tensor, was_numpy) of an array or tensor (the GPU loss kernels' operand)."""
    import torch

    if isinstance(a, torch.Tensor) and a.is_cuda:
        return a.contiguous().float(), False
    return torch.as_tensor(np.asarray(a, dtype=np.float32)).cuda(), True


def _loss_stats_block(p, g, clamp):
    """Per-class [sum p*g, sum p, sum g] plus the summed NLL of one device block (training.py
    :77-92), on the GPU (vm_loss_stats: float64 block partials, fixed-order reduction)."""
    import torch

    from . import _lib

    pd, _ = _dev(p)
    gd, _ = _dev(g)
    c = pd.shape[-1]
    rows = pd.numel() // c
    ws = torch.empty(2 * 148 * (3 * c + 1), dtype=torch.float64, device=pd.device)
    out = torch.empty(3 * c + 1, dtype=torch.float64, device=pd.device)
    _lib.call("vm_loss_stats", _lib.ptr(pd), _lib.ptr(gd), rows, c, float(clamp), _lib.ptr(ws), _lib.ptr(out),
              _lib.stream_ptr())
    return out.cpu().numpy()


def loss_stats_local(probs, onehot, clamp=1e-12):
    """Worker-level statistics of the local block (training.py:77-92) on the GPU."""
    return _loss_stats_block(probs, onehot, clamp)


@dataclass(frozen=True)
class _RunCtx:
    """The constants a step needs on the worker side (training.py:53-65)."""

    num_classes: int
    dice_classes: tuple
    w_dice: float
    w_ce: float
    clamp: float
    total_batch_voxels: int
    lr: float = 0.003
    momentum: float = 0.9
    phase_barrier: bool = True
    param_order: tuple = ()


def losses_from_stats(stats, rc):
    """(combined, dice, ce) from reduced statistics (training.py:103-107)."""
    dice = soft_dice_from_stats(stats, rc.num_classes, rc.dice_classes)
    ce = float(stats[3 * rc.num_classes]) / rc.total_batch_voxels
    return rc.w_dice * dice + rc.w_ce * ce, dice, ce


def loss_grad_local(probs, onehot, stats, rc):
    """dL/dprobs of the combined loss per voxel from the globally reduced statistics
    (training.py:110-127), on the GPU (vm_loss_grad); numpy in, numpy out."""
    import torch

    from . import _lib

    pd, was_np = _dev(probs)
    gd, _ = _dev(onehot)
    st = torch.as_tensor(np.asarray(stats, dtype=np.float64)).to(pd.device)
    c = pd.shape[-1]
    out = torch.empty_like(pd)
    mask = sum(1 << k for k in rc.dice_classes)
    _lib.call("vm_loss_grad", _lib.ptr(pd), _lib.ptr(gd), _lib.ptr(st), pd.numel() // c, c, float(rc.w_dice),
              float(rc.w_ce), float(rc.total_batch_voxels), mask, float(rc.clamp), _lib.ptr(out), _lib.stream_ptr())
    if was_np:
        return out.cpu().numpy().astype(np.asarray(probs).dtype)
    return out


def sgd_momentum_step(params, moments, grads, lr, momentum, order):
    """v <- momentum*v + g; p <- p - lr*v per parameter blob, in ``order``; layers with
    non-finite gradients are skipped and returned (training.py:202-219).  In place on the
    reference-layout dicts, through the step's fused kernel (vm_sgd_momentum, numpy's fp32
    operation order, so the results are bitwise numpy's)."""
    import torch

    from . import _lib

    keys = [(nid, k) for nid in order for k in ("kernel", "bias")]
    offs = [0]
    for nid, k in keys:
        offs.append(offs[-1] + int(np.asarray(params[nid][k]).size))
    flat = {}
    for name, store in (("p", params), ("v", moments)):
        flat[name] = torch.cat([torch.as_tensor(np.asarray(store[nid][k], np.float32)).reshape(-1)
                                for nid, k in keys]).cuda()
    flat["g"] = torch.cat([torch.as_tensor(np.asarray(grads[nid][0 if k == "kernel" else 1], np.float32)).reshape(-1)
                           for nid, k in keys]).cuda()
    # layers = (kernel, bias) pairs: one skip decision per layer (training.py:210-213)
    loffs = torch.tensor(offs[::2], dtype=torch.int64).cuda()
    nl = len(order)
    flags = torch.zeros(nl, dtype=torch.int32).cuda()
    most = max(b - a for a, b in zip(offs[::2], offs[2::2])) if nl else 0
    _lib.call("vm_sgd_momentum", _lib.ptr(flat["p"]), _lib.ptr(flat["v"]), _lib.ptr(flat["g"]), _lib.ptr(loffs), nl,
              most, _lib.ptr(flags), float(lr), float(momentum), _lib.stream_ptr())
    fl = flags.cpu().numpy()
    hp, hv = flat["p"].cpu().numpy(), flat["v"].cpu().numpy()
    for i, (nid, k) in enumerate(keys):
        a, b = offs[i], offs[i + 1]
        shape = np.asarray(params[nid][k]).shape
        params[nid][k][...] = hp[a:b].reshape(shape)
        moments[nid][k][...] = hv[a:b].reshape(shape)
    return [nid for nid, f in zip(order, fl) if f]


def soft_dice_from_stats(stats, num_classes, dice_classes, eps=DICE_EPS):
    """1 - mean over ``dice_classes`` of (2*sum(p*g)+eps)/(sum(p)+sum(g)+eps) (training.py:95-100)."""
    c = num_classes
    pg, ps, gs = stats[0:c], stats[c : 2 * c], stats[2 * c : 3 * c]
    ratios = [(2.0 * float(pg[k]) + eps) / (float(ps[k]) + float(gs[k]) + eps) for k in dice_classes]
    return 1.0 - sum(ratios) / len(ratios)


def _reduced_stats(probs, labels_onehot, clamp, tag):
    def fn(ctx, p, g):
        return ctx.all_reduce_sum(_loss_stats_block(p, g, clamp), tag=tag)

    return next(r for r in probs.mesh.run(fn, per_worker=(probs.blocks, labels_onehot.blocks)) if r is not None)


def soft_dice_loss(probs, labels_onehot, dice_classes=(1, 2)):
    """Distributed soft-Dice loss over sharded probabilities and one-hot labels (training.py:130-139)."""
    stats = _reduced_stats(probs, labels_onehot, 1e-12, "dice-stats")
    return soft_dice_from_stats(stats, probs.spec.extent("c"), dice_classes)


def cross_entropy_loss(probs, labels_onehot, clamp=1e-12):
    """Distributed mean per-voxel negative log-likelihood (training.py:142-152)."""
    c = probs.spec.extent("c")
    stats = _reduced_stats(probs, labels_onehot, clamp, "ce-stats")
    voxels = int(np.prod([e for n, e in probs.spec.dims if n != "c"]))
    return float(stats[3 * c]) / voxels


def combined_loss(weights, probs, labels_onehot, dice_classes=(1, 2)):
    """training.py:155-158."""
    return weights.dice * soft_dice_loss(probs, labels_onehot, dice_classes) + weights.ce * cross_entropy_loss(
        probs, labels_onehot
    )


# ---------------------------------------------------------------------------- metrics
def hard_dice(pred_mask, gt_mask):
    """2|A∩B| / (|A|+|B|); 1 when both are empty, 0 when only one is (training.py:166-175)."""
    a, b = int(np.count_nonzero(pred_mask)), int(np.count_nonzero(gt_mask))
    if a + b == 0:
        return 1.0
    if a == 0 or b == 0:
        return 0.0
    return 2.0 * int(np.count_nonzero(np.logical_and(pred_mask, gt_mask))) / (a + b)


def _check_pairs(preds, gts):
    if len(preds) != len(gts):
        raise VoxmeshError(f"{len(preds)} predictions vs {len(gts)} ground truths")


def dice_per_case(preds, gts, cls=2):
    """Mean over cases of the hard Dice of class ``cls`` (training.py:178-183)."""
    _check_pairs(preds, gts)
    return float(np.mean([hard_dice(p == cls, g == cls) for p, g in zip(preds, gts)]))


def dice_global(preds, gts, cls=2):
    """Hard Dice of class ``cls`` with all cases pooled (training.py:186-194)."""
    _check_pairs(preds, gts)
    inter = tot = 0
    for p, g in zip(preds, gts):
        pm, gm = p == cls, g == cls
        inter += int(np.count_nonzero(pm & gm))
        tot += int(np.count_nonzero(pm)) + int(np.count_nonzero(gm))
    return 1.0 if tot == 0 else 2.0 * inter / tot


# ---------------------------------------------------------------------------- checkpoints
def save_checkpoint(path, step, params, moments, extra=None):
    """Reference checkpoint layout (training.py:414-428)."""
    path = Path(path)
    path.mkdir(parents=True, exist_ok=True)
    names = []
    for kind, store in (("param", params), ("moment", moments)):
        for nid, blobs in store.items():
            for key, arr in blobs.items():
                name = f"{kind}__{nid}__{key}.npy"
                np.save(path / name, np.asarray(arr))
                names.append(name)
    manifest = {"step": int(step), "blobs": names}
    manifest.update(extra or {})
    (path / "manifest.json").write_text(json.dumps(manifest, indent=2, default=str))


def load_checkpoint(path):
    """(step, params, moments) from a reference-format checkpoint (training.py:431-439)."""
    path = Path(path)
    manifest = json.loads((path / "manifest.json").read_text())
    stores = {"param": {}, "moment": {}}
    for name in manifest["blobs"]:
        kind, nid, key = name[: -len(".npy")].split("__")
        if kind not in stores:
            raise VoxmeshError(f"checkpoint {path}: unknown blob kind in {name!r}")
        stores[kind].setdefault(nid, {})[key] = np.load(path / name)
    return manifest["step"], stores["param"], stores["moment"]


# ---------------------------------------------------------------------------- batches
def _image_labels(rec):
    if hasattr(rec, "image"):
        return rec.image, rec.labels
    return rec[0], rec[1]


class BatchSource:
    """Deterministic batches from (seed, step) (training.py:241-279): epoch e visits the
    records in ``default_rng(SeedSequence([seed, 7919, e])).permutation(n)`` order.
    Returns the host image ``[B, E, E, E, 1]`` (f32) and labels ``[B, E, E, E]`` (u8); the
    one-hot expansion happens on the GPU."""

    def __init__(self, records, batch_size, seed, augment=None):
        if not records:
            raise VoxmeshError("empty training set")
        self.records = list(records)
        self.batch_size = int(batch_size)
        self.seed = int(seed)
        self.augment = augment
        self._perms = {}

    def perm(self, epoch):
        if epoch not in self._perms:
            rng = np.random.default_rng(np.random.SeedSequence([self.seed, 7919, int(epoch)]))
            self._perms[epoch] = rng.permutation(len(self.records))
        return self._perms[epoch]

    def record_index(self, global_idx):
        n = len(self.records)
        return int(self.perm(global_idx // n)[global_idx % n])

    def _pair(self, global_idx):
        rec = self.records[self.record_index(global_idx)]
        img, lab = _image_labels(rec)
        if self.augment is not None:  # training.py:268-272
            from . import augment as _aug

            aug_seed = int(np.random.SeedSequence([self.seed, 104729, int(global_idx)]).generate_state(1)[0])
            out = _aug.augment_pipeline(_aug.VolumeRecord(img, lab, getattr(rec, "id", "")),
                                        _aug.with_seed(self.augment, aug_seed))
            img, lab = out.image, out.labels
        return img, lab

    def batch(self, step):
        pairs = [self._pair(step * self.batch_size + j) for j in range(self.batch_size)]
        img = np.stack([np.asarray(p[0], dtype=np.float32) for p in pairs])[..., None]
        lab = np.stack([np.asarray(p[1], dtype=np.uint8) for p in pairs])
        return img, lab


# ---------------------------------------------------------------------------- placement
def _batch_axis(graph):
    return graph.layout.axis_for("batch") if graph.layout is not None else None


def _spatial_axes(graph):
    if graph.layout is None:
        return []
    return [a for a in (graph.layout.axis_for(d) for d in ("x", "y", "z")) if a is not None]


def _blocks(graph, arr, spatial_from=1):
    """Per-rank local blocks of a host array ``[B, X, Y, Z, ...]``: dim 0 split over the
    layout's batch axis, the spatial dims (from ``spatial_from``) over theirs — the block
    slices of sharding.local_slices (sharding.py:123-143)."""
    mesh, layout = graph.mesh, graph.layout
    out = []
    for coord in mesh.coords:
        sl = [slice(None)] * arr.ndim
        for i, d in enumerate(("batch", "x", "y", "z")):
            ax = layout.axis_for(d) if layout is not None else None
            if ax is None:
                continue
            dim = 0 if d == "batch" else spatial_from + i - 1
            size = mesh.axis_size(ax)
            if arr.shape[dim] % size:
                raise ShardingError(f"dim {d!r} of extent {arr.shape[dim]} is not divisible by mesh axis "
                                    f"{ax!r} of size {size}")
            n = arr.shape[dim] // size
            c = coord[mesh.axis_index[ax]]
            sl[dim] = slice(c * n, (c + 1) * n)
        out.append(np.ascontiguousarray(arr[tuple(sl)]))
    return out


def _make_steps(graph, params, cfg, batch, key="vm_step", evaluation=False):
    """One UNetStep per rank: the local batch is ``batch`` over the layout's batch axis; the
    loss is normalised by the global batch (training.py:396-406).  ``evaluation``: batch of one
    sample per batch coordinate, per-sample statistics summed over the spatial axes only and
    normalised by one volume (training.py:346-355, :557-561), argmax predictions kept."""
    import torch

    from .step import UNetStep

    mesh = graph.mesh
    b_axis = _batch_axis(graph)
    bdiv = mesh.axis_size(b_axis) if b_axis else 1
    if batch % bdiv:
        raise ShardingError(f"batch {batch} is not divisible by mesh axis {b_axis!r} of size {bdiv}")
    dtype = torch.bfloat16 if cfg.compute_dtype == "bf16" else torch.float32
    E = graph.config.input_extent
    multi = mesh.worker_count > 1
    spatial = _spatial_axes(graph)

    def make(ctx):
        st = UNetStep(graph, params, batch=batch // bdiv, ctx=ctx if multi else None, device=ctx.device, dtype=dtype,
                      lr=cfg.lr, momentum=cfg.momentum,
                      loss_weights=(cfg.loss_weights.dice, cfg.loss_weights.ce),
                      dice_classes=tuple(cfg.dice_classes), clamp=cfg.prob_clamp, global_shape=(E, E, E),
                      global_batch=1 if evaluation else batch)
        if evaluation:
            st.keep_pred = True
            st.stats_axes = tuple(spatial)
        if (multi and st.comm is not None and st.has_halo and max(st.halo.nbr6[2:]) < 0
                and os.environ.get("VOXMESH_HALO", "peer") == "peer"):
            # depth-only split over NCCL ranks: the peer-memory halo fused into the conv kernels
            # (every rank falls back to NCCL together if a CUDA-IPC mapping fails)
            try:
                st.use_peer_halo()
            except HaloError:
                pass
        ctx.store[key] = st
        return None

    mesh.run(make)


def _zero_moments(params):
    return {n: {k: np.zeros_like(np.asarray(v)) for k, v in b.items()} for n, b in params.items()}


def install_params(graph, params, moments=None):
    """Put an externally built parameter store on every rank (training.py:536-540): builds
    the per-rank steps when none exist yet; ``moments=None`` resets momentum to zero."""
    have = graph.mesh.run(lambda ctx: "vm_step" in ctx.store)[0]
    if not have:
        b_axis = _batch_axis(graph)
        _make_steps(graph, params, TrainConfig(), graph.mesh.axis_size(b_axis) if b_axis else 1)
    mom = moments if moments is not None else _zero_moments(params)
    graph.mesh.run(lambda ctx: ctx.store["vm_step"].load_state(params, mom))
    graph.mesh.run(lambda ctx: ctx.store.pop("vm_eval_step", None) and None)


def _export_state(graph):
    return graph.mesh.run(lambda ctx: (ctx.store["vm_step"].param_dict(), ctx.store["vm_step"].moment_dict())
                          if ctx.rank == 0 else None)[0]


def _launch(ctx, img, lab):
    st = ctx.store["vm_step"]
    return st.launch_host_step(img, lab, replay=ctx.store.get("vm_graph_replay"))


def _collect(ctx, handle):
    return ctx.store["vm_step"].collect(handle)


def _capture(ctx):
    g = ctx.store["vm_step"].capture()
    ctx.store["vm_graph"] = g
    ctx.store["vm_graph_replay"] = g.replay if g is not None else None
    return g is not None


def train_loop(graph, dataset, cfg, resume_from=None, run_echo=None):
    """Train on the graph's mesh; returns the final TrainState (training.py:442-533)."""
    from . import unet as _unet

    records = dataset.load_split("train") if hasattr(dataset, "load_split") else list(dataset)
    mesh = graph.mesh
    if resume_from is not None:
        start, params, moments = load_checkpoint(resume_from)
    else:
        start = 0
        params = _unet.init_params(graph, cfg.seed)
        moments = None
    _make_steps(graph, params, cfg, cfg.batch_size)
    if moments is not None:
        install_params(graph, None, moments)

    out_dir = Path(cfg.out_dir) if cfg.out_dir else None
    csv_f = None
    if out_dir:
        out_dir.mkdir(parents=True, exist_ok=True)
        echo = {
            "mesh": mesh.describe(), "layout": graph.layout.as_dict() if graph.layout is not None else {},
            "seed": cfg.seed, "steps": cfg.steps, "batch_size": cfg.batch_size, "lr": cfg.lr,
            "momentum": cfg.momentum, "dtype": cfg.dtype, "compute_dtype": cfg.compute_dtype,
            "dice_classes": list(cfg.dice_classes), "loss_weights": [cfg.loss_weights.dice, cfg.loss_weights.ce],
            "augment": bool(cfg.augment), "config_kv": graph.config.to_kv(),
            "resume_from": str(resume_from) if resume_from else None,
        }
        echo.update(run_echo or {})
        (out_dir / "run.json").write_text(json.dumps(echo, indent=2, default=str))
        fresh = resume_from is None or not (out_dir / "metrics.csv").exists()
        csv_f = open(out_dir / "metrics.csv", "w" if fresh else "a")
        if fresh:
            csv_f.write("step,loss,dice_loss,ce_loss,lr,wall_ms\n")

    source = BatchSource(records, cfg.batch_size, cfg.seed, cfg.augment)
    state = TrainState(start, params, moments or {})
    # step k+1's host batch is built while step k runs on the GPU; step k's loss is read one
    # step behind (async D2H into pinned memory), so the loop never waits on a loss it does
    # not need yet.  The step is a captured CUDA graph whenever the transport allows it.
    pending = None

    def finish(item):
        step, t0, handles = item
        (loss, dice, ce), skipped = mesh.run(_collect, per_worker=(handles,))[0]
        wall_ms = (time.perf_counter() - t0) * 1e3
        if skipped:
            warnings.warn(f"step {step}: non-finite gradients, skipped layers {skipped}")
        state.step = step + 1
        state.history.append((step, loss, dice, ce, wall_ms))
        if csv_f:
            csv_f.write(f"{step},{loss:.8f},{dice:.8f},{ce:.8f},{cfg.lr},{wall_ms:.2f}\n")
        if cfg.log_every and step % cfg.log_every == 0:
            print(f"step {step:5d}  loss {loss:.6f}  dice {dice:.6f}  ce {ce:.6f}  ({wall_ms:.0f} ms)")
        if cfg.checkpoint_every and out_dir and (step + 1) % cfg.checkpoint_every == 0:
            p, m = _export_state(graph)
            save_checkpoint(out_dir / "checkpoints" / f"step_{step + 1:06d}", step + 1, p, m,
                            extra={"config_kv": graph.config.to_kv(), "seed": cfg.seed})

    try:
        for step in range(start, start + cfg.steps):
            img, lab = source.batch(step)
            t0 = time.perf_counter()
            cur = (step, t0, mesh.run(_launch, per_worker=(_blocks(graph, img), _blocks(graph, lab))))
            if pending is not None:
                finish(pending)
                pending = None
            ckpt = cfg.checkpoint_every and out_dir and (step + 1) % cfg.checkpoint_every == 0
            if step == start or ckpt:  # a checkpoint must not see the next step's update
                finish(cur)
                if step == start:  # the first step ran eagerly; later ones replay its graph
                    mesh.run(_capture)
            else:
                pending = cur
        if pending is not None:
            finish(pending)
    finally:
        if csv_f:
            csv_f.close()
    state.params, state.moments = _export_state(graph)
    if out_dir:
        save_checkpoint(out_dir / "checkpoints" / f"step_{state.step:06d}", state.step, state.params,
                        state.moments, extra={"config_kv": graph.config.to_kv(), "seed": cfg.seed})
    return state


def _eval_chunk(ctx, img, lab):
    """Forward of one sample block; per-sample loss statistics and hard-Dice counts summed
    over the spatial axes (training.py:346-355).  Predictions stay on the GPU: the argmax is
    written by the head kernel and counted against the labels by vm_label_counts."""
    import torch

    from . import _lib

    st = ctx.store["vm_eval_step"]
    st.upload(torch.from_numpy(img), torch.from_numpy(lab))
    st.forward()
    counts = torch.zeros(3 * st.ncls, dtype=torch.int64, device=st.device)
    _lib.call("vm_label_counts", _lib.ptr(st.pred), _lib.ptr(st.labels), st.nvox, st.ncls, _lib.ptr(counts),
              _lib.stream_ptr())
    if st.stats_axes:
        counts = ctx.all_reduce_sum(counts, axes=list(st.stats_axes), tag="eval-counts")
    st._check_labels(int(st.label_err.item()))
    return st.stats.double().cpu().numpy(), counts.cpu().numpy()


def _dice_from_counts(inter, a, b):
    """hard_dice (training.py:166-175) from |A∩B|, |A|, |B|."""
    if a + b == 0:
        return 1.0
    if a == 0 or b == 0:
        return 0.0
    return 2.0 * inter / (a + b)


def evaluate(graph, dataset, cfg, params=None, cls=2):
    """Forward-only pass over records on the GPU (training.py:543-602): records go in chunks
    of the batch axis' width, a partial last chunk is padded by repeating its last record and
    the padding is dropped; returns hard Dice of class ``cls`` per case and pooled, and the
    mean per-sample loss.  ``params`` defaults to the weights of the last ``train_loop`` /
    ``install_params`` on this graph."""
    records = dataset.load_split("val") if hasattr(dataset, "load_split") else list(dataset)
    if not records:
        raise VoxmeshError("empty evaluation set")
    mesh = graph.mesh
    b_axis = _batch_axis(graph)
    chunk = mesh.axis_size(b_axis) if b_axis else 1
    have = mesh.run(lambda ctx: "vm_step" in ctx.store)[0]
    if params is None and not have:
        raise VoxmeshError("evaluate: no parameters installed on this graph")
    if mesh.run(lambda ctx: "vm_eval_step" in ctx.store)[0] is False:
        _make_steps(graph, params if params is not None else _export_state(graph)[0], cfg, chunk,
                    key="vm_eval_step", evaluation=True)
    if params is not None:
        mesh.run(lambda ctx: ctx.store["vm_eval_step"].load_state(params))
    else:  # the training step's current weights
        def sync(ctx):
            ev = ctx.store["vm_eval_step"]
            ev.params.copy_(ctx.store["vm_step"].params)
            ev.repack()
        mesh.run(sync)
    ncls = graph.config.num_classes
    E = graph.config.input_extent
    dice_cases, losses = [], []
    inter_t = a_t = b_t = 0
    for i0 in range(0, len(records), chunk):
        recs = records[i0 : i0 + chunk]
        valid = len(recs)
        while len(recs) < chunk:
            recs.append(recs[-1])
        pairs = [_image_labels(r) for r in recs]
        img = np.stack([np.asarray(p[0], dtype=np.float32) for p in pairs])[..., None]
        lab = np.stack([np.asarray(p[1], dtype=np.uint8) for p in pairs])
        res = mesh.run(_eval_chunk, per_worker=(_blocks(graph, img), _blocks(graph, lab)))
        by_sample = {}
        for rank, coord in enumerate(mesh.coords):
            bc = coord[mesh.axis_index[b_axis]] if b_axis else 0
            by_sample.setdefault(bc, res[rank])
        for j in range(valid):
            stats, counts = by_sample[j]
            inter, a, b = int(counts[cls]), int(counts[ncls + cls]), int(counts[2 * ncls + cls])
            dice_cases.append(_dice_from_counts(inter, a, b))
            inter_t, a_t, b_t = inter_t + inter, a_t + a, b_t + b
            ds = soft_dice_from_stats(stats, ncls, tuple(cfg.dice_classes))
            losses.append(cfg.loss_weights.dice * ds + cfg.loss_weights.ce * float(stats[3 * ncls]) / E ** 3)
    return {
        "dice_per_case": float(np.mean(dice_cases)),
        "dice_global": 1.0 if a_t + b_t == 0 else 2.0 * inter_t / (a_t + b_t),
        "mean_loss": float(sum(losses) / len(losses)),
        "n_cases": len(dice_cases),
    }
