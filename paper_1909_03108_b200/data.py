"""Synthetic CT-like volumes: the input specification of the benchmark.

Same distribution and random-stream consumption as the reference generator
``data_io.synthesize_record`` (data_io.py:163-184) with record seeds
``SeedSequence([seed, i])`` (data_io.py:196): background N(0, 0.1), one liver
ellipsoid (centre E/2 +- U(E/10), radii U(0.30, 0.40) E, +1.0, label 1),
1-3 tumour spheres (radius U(E/16, E/8), centred on liver voxels, clipped to
the liver, +1.5, label 2).  Draw order is identical, so records are bitwise the
reference's (checked in tests/test_host_logic.py::test_synthetic_record_bitwise_reference).
"""

from __future__ import annotations

import numpy as np


def _inside(shape, center, radii):
    """Boolean ellipsoid mask; sum of squared normalised offsets <= 1 (float64)."""
    axes = [((np.arange(n, dtype=np.float64) - c) / r) ** 2 for n, c, r in zip(shape, center, radii)]
    q = axes[0][:, None, None] + axes[1][None, :, None]
    q = q + axes[2][None, None, :]
    return q <= 1.0


def synth_record(extent, seed=7, index=0):
    """(image f32 [E,E,E], labels u8 [E,E,E]) of record ``index`` of a dataset seeded ``seed``."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), int(index)]))
    e = int(extent)
    shape = (e, e, e)
    image = rng.normal(0.0, 0.1, shape)
    center = [e / 2 + rng.uniform(-e / 10, e / 10) for _ in range(3)]
    radii = [rng.uniform(0.30, 0.40) * e for _ in range(3)]
    liver = _inside(shape, center, radii)
    labels = liver.astype(np.uint8)
    image += liver
    pts = np.argwhere(liver)
    tumour = np.zeros(shape, dtype=bool)
    for _ in range(int(rng.integers(1, 4))):
        c = pts[rng.integers(len(pts))]
        r = rng.uniform(e / 16, e / 8)
        tumour |= _inside(shape, c, (r, r, r))
    tumour &= liver
    labels[tumour] = 2
    image = image + 1.5 * tumour
    return image.astype(np.float32), labels


def synth_batch(extent, batch, seed=7, start=0):
    """[B, E, E, E, 1] f32 images and [B, E, E, E] u8 labels."""
    recs = [synth_record(extent, seed, start + i) for i in range(batch)]
    return np.stack([r[0] for r in recs])[..., None], np.stack([r[1] for r in recs])
