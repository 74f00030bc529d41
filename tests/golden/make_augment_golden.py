"""Generate the augmentation fixtures from the REFERENCE implementation (build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_augment_golden.py

``augment_golden.npz``: for each case, the input record (image f32, labels u8), the
SynthConfig fields and the reference ``augment_pipeline`` output (augment.py:137-151):
* ``ct``: the CT-like 16^3 record of the reference tests (integer intensities), blur 1.5;
* ``synth``: ``data_io.synthesize_record(32, ...)`` (float intensities), blur 1.5, 1-3 tumours;
* ``sharp``: the same record, blur 0 (exact mask shift);
* ``free``: a tumour-free record with ``default_delta``.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def ct_like_record(seed, extent=16):
    rng = np.random.default_rng(seed)
    labels = np.zeros((extent,) * 3, np.uint8)
    c = extent // 2
    r = extent // 3
    g = np.ogrid[:extent, :extent, :extent]
    liver = sum(((gi - c) / r) ** 2 for gi in g) <= 1.0
    labels[liver] = 1
    tumor = sum(((gi - c) / (r // 2)) ** 2 for gi in g) <= 1.0
    labels[tumor & liver] = 2
    image = rng.integers(-100, 100, (extent,) * 3).astype(np.float32)
    image[labels == 1] += 80
    image[labels == 2] += 120
    return image, labels


def main():
    sys.path.insert(0, REF)
    from voxmesh import augment, data_io

    cases = {}
    img, lab = ct_like_record(1)
    cases["ct"] = (img, lab, dict(seed=5, blur_sigma=1.5))
    rec = data_io.synthesize_record(32, np.random.default_rng(np.random.SeedSequence([7, 2])), "s")
    cases["synth"] = (rec.image, rec.labels, dict(seed=9, blur_sigma=1.5))
    cases["sharp"] = (rec.image, rec.labels, dict(seed=3, blur_sigma=0.0))
    free_lab = rec.labels.copy()
    free_lab[free_lab == 2] = 1
    cases["free"] = (rec.image, free_lab, dict(seed=11, blur_sigma=1.5, default_delta=0.75, n_tumors=(2, 3)))
    out = {}
    for name, (img, lab, kw) in cases.items():
        cfg = augment.SynthConfig(**kw)
        res = augment.augment_pipeline(data_io.VolumeRecord(img.copy(), lab.copy(), name), cfg)
        out[f"{name}_image"] = img
        out[f"{name}_labels"] = lab
        out[f"{name}_out_image"] = res.image
        out[f"{name}_out_labels"] = res.labels
        out[f"{name}_cfg"] = np.array([kw.get("seed", 0), kw.get("blur_sigma", 1.5),
                                       kw.get("default_delta", np.nan), *kw.get("n_tumors", (1, 3))])
    np.savez_compressed(os.path.join(HERE, "augment_golden.npz"), **out)
    print("wrote augment_golden.npz:", sorted(cases))


if __name__ == "__main__":
    main()
