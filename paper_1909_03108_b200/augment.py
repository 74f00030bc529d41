"""Tumour remove / synthesise augmentation on the GPU — the reference ``voxmesh.augment``
API (augment.py:1-155) over device kernels (``csrc/augment.cu``).

The pipeline measures the mean intensity difference between tumour and healthy liver,
removes the real tumour, then paints new ones: random ellipsoids inside the liver, shifted
by the measured (1/256-quantised) delta, with optionally Gaussian-blurred boundaries.
Background voxels are never touched.  The random draws (tumour count, centres, radii) and
the Gaussian weights are made on the host with numpy exactly as the reference makes them;
everything per-voxel runs on the GPU:

* ``vm_aug_stats``: the tumour / liver float64 sums of ``intensity_delta`` (augment.py:53-64);
  the GPU summation order differs from numpy's pairwise sum in the last bits, which the
  1/256 quantisation (``quantize_delta``) absorbs;
* ``vm_aug_remove`` (augment.py:67-78);
* ``vm_aug_count_chunks``: liver-voxel counts per chunk, so the host can locate the k-th
  liver voxel in ``np.argwhere`` order without copying the labels;
* ``vm_aug_paint`` / ``vm_aug_blur_axis`` / ``vm_aug_finish``: the ellipsoid union (float64,
  the reference's accumulation order), ``scipy.ndimage.gaussian_filter`` (mode constant,
  truncate 4: one correlate1d pass per axis with scipy's symmetric-kernel order in double,
  rounded to f32) and the final clip / mask / shift / relabel (augment.py:119-133).

Records are ``VolumeRecord(image f32 [D,H,W], labels u8 [D,H,W], id)`` as in the reference
(data_io.py); ``*_device`` variants take and return CUDA tensors.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .errors import AugmentError

DELTA_STEP = 1.0 / 256.0
_CHUNK = 4096


@dataclass
class VolumeRecord:
    """(image f32, labels u8, id) — data_io.VolumeRecord."""

    image: np.ndarray
    labels: np.ndarray
    id: str = ""


@dataclass(frozen=True)
class SynthConfig:
    """How synthetic tumours are drawn: count range, per-axis radii, blur, seed (augment.py:30-45)."""

    n_tumors: tuple = (1, 3)
    radius_range: tuple = (2.5, 4.5)
    blur_sigma: float = 1.5
    seed: int = 0
    label_threshold: float = 0.5
    default_delta: float | None = None

    def __post_init__(self):
        if self.n_tumors[0] < 1 or self.n_tumors[1] < self.n_tumors[0]:
            raise AugmentError(f"bad tumor count range {self.n_tumors}")
        if self.radius_range[0] < 1.0:
            raise AugmentError(f"radii must be >= 1 voxel, got {self.radius_range}")


def quantize_delta(delta):
    """Snap an intensity shift to 1/256 steps (augment.py:48-50)."""
    return float(np.float32(round(delta / DELTA_STEP) * DELTA_STEP))


def with_seed(cfg, seed):
    return replace(cfg, seed=int(seed))


# ---------------------------------------------------------------------------- device ops
def _torch():
    import torch

    return torch


def _to_device(rec):
    torch = _torch()
    img = torch.from_numpy(np.ascontiguousarray(rec.image, dtype=np.float32)).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(rec.labels, dtype=np.uint8)).cuda()
    return img, lab


def _to_record(img, lab, rid):
    return VolumeRecord(img.cpu().numpy(), lab.cpu().numpy(), rid)


def stats_device(image, labels):
    """(sum image | tumour, #tumour, sum image | liver, #liver) as Python floats (float64)."""
    torch = _torch()
    ws = torch.empty(_lib.call_size("vm_aug_stats_ws_bytes") // 8, dtype=torch.float64, device=image.device)
    out = torch.empty(4, dtype=torch.float64, device=image.device)
    _lib.call("vm_aug_stats", _lib.ptr(image), _lib.ptr(labels), image.numel(), _lib.ptr(ws), _lib.ptr(out),
              _lib.stream_ptr())
    return [float(v) for v in out.cpu().numpy()]


def intensity_delta_device(image, labels, rid=""):
    st, ct, sl, cl = stats_device(image, labels)
    if ct == 0:
        raise AugmentError(f"{rid}: no tumor voxels to measure")
    if cl == 0:
        raise AugmentError(f"{rid}: no non-tumor liver voxels to measure")
    return st / ct - sl / cl


def remove_tumor_device(image, labels, delta):
    """In place: image[tumour] -= f32(delta); labels[tumour] = 1."""
    _lib.call("vm_aug_remove", _lib.ptr(image), _lib.ptr(labels), image.numel(), float(np.float32(delta)),
              _lib.stream_ptr())


def _liver_index(labels, counts_cum, k):
    """Flat index of the k-th liver voxel in C order (np.argwhere(labels == 1)[k])."""
    ch = int(np.searchsorted(counts_cum, k, side="right"))
    before = int(counts_cum[ch - 1]) if ch > 0 else 0
    seg = labels[ch * _CHUNK:(ch + 1) * _CHUNK].cpu().numpy()
    pos = np.flatnonzero(seg == 1)[k - before]
    return ch * _CHUNK + int(pos)


def synthesize_tumor_device(image, labels, delta, cfg, rid=""):
    """In place on device tensors image f32 [D,H,W] / labels u8 [D,H,W] (augment.py:89-134)."""
    torch = _torch()
    dev = image.device
    shape = tuple(labels.shape)
    n = labels.numel()
    counts = torch.empty((n + _CHUNK - 1) // _CHUNK, dtype=torch.int32, device=dev)
    flat = labels.reshape(-1)
    _lib.call("vm_aug_count_chunks", _lib.ptr(flat), n, _CHUNK, 2, _lib.ptr(counts), _lib.stream_ptr())
    if int(counts.sum().item()) > 0:
        raise AugmentError(f"{rid}: record already has tumor; remove it first")
    _lib.call("vm_aug_count_chunks", _lib.ptr(flat), n, _CHUNK, 1, _lib.ptr(counts), _lib.stream_ptr())
    cum = np.cumsum(counts.cpu().numpy().astype(np.int64))
    nliver = int(cum[-1])
    if nliver == 0:
        raise AugmentError(f"{rid}: empty liver, nowhere to synthesize")
    rng = np.random.default_rng(cfg.seed)
    ntum = int(rng.integers(cfg.n_tumors[0], cfg.n_tumors[1] + 1))
    centers, radii = [], []
    for _ in range(ntum):
        # the centre is a liver voxel and every radius is >= 1, so the first draw's ball is
        # never empty: the reference's retry loop (augment.py:105-112) never draws again
        k = int(rng.integers(nliver))
        centers.append(np.unravel_index(_liver_index(flat, cum, k), shape))
        radii.append(rng.uniform(cfg.radius_range[0], cfg.radius_range[1], 3))
    c_t = torch.from_numpy(np.asarray(centers, dtype=np.int64).reshape(-1)).to(dev)
    r_t = torch.from_numpy(np.asarray(radii, dtype=np.float64).reshape(-1)).to(dev)
    mask = torch.empty(shape, dtype=torch.float32, device=dev)
    _lib.call("vm_aug_paint", _lib.ptr(flat), shape[0], shape[1], shape[2], _lib.ptr(c_t), _lib.ptr(r_t), ntum,
              _lib.ptr(mask), _lib.stream_ptr())
    w = mask
    if cfg.blur_sigma > 0:
        # scipy.ndimage.gaussian_filter1d: radius int(truncate*sigma + 0.5), weights
        # exp(-0.5/sigma^2 * x^2) / sum in float64 (_gaussian_kernel1d), computed with numpy
        sd = float(cfg.blur_sigma)
        rad = int(4.0 * sd + 0.5)
        x = np.arange(-rad, rad + 1)
        phi = np.exp(-0.5 / (sd * sd) * x ** 2)
        phi = phi / phi.sum()
        wk = torch.from_numpy(np.ascontiguousarray(phi[rad:], dtype=np.float64)).to(dev)
        tmp = torch.empty_like(mask)
        src, dst = mask, tmp
        for axis in range(3):
            _lib.call("vm_aug_blur_axis", _lib.ptr(src), _lib.ptr(dst), shape[0], shape[1], shape[2], axis,
                      _lib.ptr(wk), rad, _lib.stream_ptr())
            src, dst = dst, src
        w = src
    _lib.call("vm_aug_finish", _lib.ptr(image), _lib.ptr(flat), _lib.ptr(w), n, float(np.float32(delta)),
              float(cfg.label_threshold), _lib.stream_ptr())
    _lib.call("vm_aug_count_chunks", _lib.ptr(flat), n, _CHUNK, 2, _lib.ptr(counts), _lib.stream_ptr())
    if int(counts.sum().item()) == 0:
        warnings.warn(
            f"{rid}: synthetic tumor vanished below the label threshold "
            f"(radii {cfg.radius_range} too small for sigma {cfg.blur_sigma})"
        )


def augment_pipeline_device(image, labels, cfg, rid=""):
    """Measure delta, remove the real tumour, synthesise new ones (augment.py:137-151), in place."""
    torch = _torch()
    flat = labels.reshape(-1)
    counts = torch.empty((flat.numel() + _CHUNK - 1) // _CHUNK, dtype=torch.int32, device=labels.device)
    _lib.call("vm_aug_count_chunks", _lib.ptr(flat), flat.numel(), _CHUNK, 2, _lib.ptr(counts), _lib.stream_ptr())
    if int(counts.sum().item()) > 0:
        delta = intensity_delta_device(image, labels, rid)
    elif cfg.default_delta is not None:
        delta = cfg.default_delta
    else:
        raise AugmentError(f"{rid}: tumor-free record and no default_delta configured")
    delta = quantize_delta(delta)
    remove_tumor_device(image, labels, delta)
    synthesize_tumor_device(image, labels, delta, cfg, rid)


# ---------------------------------------------------------------------------- record API
def _rec_id(rec):
    return getattr(rec, "id", "")


def intensity_delta(rec):
    """mean(image | tumour) - mean(image | healthy liver) (augment.py:53-64)."""
    img, lab = _to_device(rec)
    return intensity_delta_device(img, lab, _rec_id(rec))


def remove_tumor(rec, delta):
    """Subtract ``delta`` on tumour voxels and relabel them as liver (augment.py:67-78)."""
    img, lab = _to_device(rec)
    remove_tumor_device(img, lab, delta)
    return _to_record(img, lab, _rec_id(rec))


def synthesize_tumor(rec, delta, cfg):
    """Paint random tumours inside the liver of a tumour-free record (augment.py:89-134)."""
    img, lab = _to_device(rec)
    synthesize_tumor_device(img, lab, delta, cfg, _rec_id(rec))
    return _to_record(img, lab, _rec_id(rec))


def augment_pipeline(rec, cfg):
    """Measure delta, remove the real tumour, synthesise new ones (augment.py:137-151)."""
    img, lab = _to_device(rec)
    augment_pipeline_device(img, lab, cfg, _rec_id(rec))
    return _to_record(img, lab, _rec_id(rec))
