"""GPU tumour remove / synthesise augmentation against the reference's
own outputs (tests/golden/augment_golden.npz, made by tests/golden/make_augment_golden.py
from voxmesh.augment) — bitwise — plus the reference test properties (test_augment.py)."""

import os

import numpy as np
import pytest

from paper_1909_03108_b200 import augment as A
from paper_1909_03108_b200.errors import AugmentError

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "augment_golden.npz"))


@pytest.mark.parametrize("case", ["ct", "synth", "sharp", "free"])
def test_pipeline_bitwise_equals_reference(case):
    seed, sigma, dd, n0, n1 = GOLD[f"{case}_cfg"]
    cfg = A.SynthConfig(seed=int(seed), blur_sigma=float(sigma), n_tumors=(int(n0), int(n1)),
                        default_delta=None if np.isnan(dd) else float(dd))
    rec = A.VolumeRecord(GOLD[f"{case}_image"].copy(), GOLD[f"{case}_labels"].copy(), case)
    out = A.augment_pipeline(rec, cfg)
    assert np.array_equal(out.labels, GOLD[f"{case}_out_labels"])
    assert np.array_equal(out.image.view(np.uint32), GOLD[f"{case}_out_image"].view(np.uint32))


def test_background_never_touched_and_same_seed_identical():
    img, lab = GOLD["synth_image"], GOLD["synth_labels"]
    cfg = A.SynthConfig(seed=4)
    a = A.augment_pipeline(A.VolumeRecord(img.copy(), lab.copy(), "a"), cfg)
    b = A.augment_pipeline(A.VolumeRecord(img.copy(), lab.copy(), "b"), cfg)
    bg = lab == 0
    assert np.array_equal(a.image[bg].view(np.uint32), img[bg].view(np.uint32))
    assert (a.labels[bg] == 0).all()
    assert np.array_equal(a.image, b.image) and np.array_equal(a.labels, b.labels)


def test_sigma0_roundtrip_restores_image():
    # remove at the quantised delta, synthesise, remove again: the synthetic tumour shift is
    # exactly undone (augment.py module docstring)
    img, lab = GOLD["ct_image"], GOLD["ct_labels"]
    cfg = A.SynthConfig(seed=2, blur_sigma=0.0)
    rec = A.VolumeRecord(img.copy(), lab.copy(), "ct")
    delta = A.quantize_delta(A.intensity_delta(rec))
    cleaned = A.remove_tumor(rec, delta)
    synth = A.synthesize_tumor(cleaned, delta, cfg)
    back = A.remove_tumor(synth, delta)
    assert np.array_equal(back.image, cleaned.image)


def test_errors():
    img, lab = GOLD["ct_image"], GOLD["ct_labels"]
    with pytest.raises(AugmentError):
        A.synthesize_tumor(A.VolumeRecord(img, lab, "x"), 1.0, A.SynthConfig())  # tumour present
    free = lab.copy()
    free[free == 2] = 1
    with pytest.raises(AugmentError):
        A.intensity_delta(A.VolumeRecord(img, free, "x"))
    with pytest.raises(AugmentError):
        A.augment_pipeline(A.VolumeRecord(img, free, "x"), A.SynthConfig())  # no default_delta


def test_train_loop_with_augmentation_matches_reference_batches(tmp_path):
    # BatchSource with a SynthConfig: each sample is augmented with the reference's per-sample
    # seed; the loop runs and records it
    import paper_1909_03108_b200 as vm
    img, lab = GOLD["synth_image"], GOLD["synth_labels"]
    recs = [A.VolumeRecord(img, lab, "r0")]
    src = vm.BatchSource(recs, 1, 3, augment=A.SynthConfig(seed=0))
    bimg, blab = src.batch(0)
    seed0 = int(np.random.SeedSequence([3, 104729, 0]).generate_state(1)[0])
    ref = A.augment_pipeline(A.VolumeRecord(img.copy(), lab.copy(), "r0"), A.with_seed(A.SynthConfig(), seed0))
    assert np.array_equal(bimg[0, ..., 0], ref.image) and np.array_equal(blab[0], ref.labels)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(vm.UNetConfig(32, (8, 16), convs_per_block=1), mesh, {})
    st = vm.train_loop(graph, recs, vm.TrainConfig(steps=2, batch_size=1, out_dir=str(tmp_path),
                                                    augment=A.SynthConfig(seed=0)))
    mesh.shutdown()
    assert st.step == 2
    import json
    assert json.loads((tmp_path / "run.json").read_text())["augment"] is True
