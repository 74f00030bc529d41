"""Host-side training-loop pieces against the reference's own outputs (no GPU):
checkpoint format (a checkpoint written by voxmesh.training.save_checkpoint is committed
under tests/golden/ref_checkpoint), the deterministic batch order, and the hard-Dice
metrics (known answers from the reference's test_training.py:111-152)."""

import json
import os

import numpy as np
import pytest

import paper_1909_03108_b200 as vm
from paper_1909_03108_b200.errors import VoxmeshError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _small_graph():
    mesh = vm.create_mesh([("one", 1)], devices=["cpu"])
    return mesh, vm.build(vm.UNetConfig(8, (4, 8), convs_per_block=1), mesh, {})


def test_reads_reference_checkpoint():
    mesh, graph = _small_graph()
    step, params, moments = vm.load_checkpoint(os.path.join(GOLD, "ref_checkpoint"))
    mesh.shutdown()
    assert step == 7
    mine = vm.init_params(graph, 1)
    assert set(params) == set(mine)
    for nid in mine:
        for key in ("kernel", "bias"):
            assert np.array_equal(params[nid][key], mine[nid][key])
            assert np.all(moments[nid][key] == 0.5) and moments[nid][key].dtype == mine[nid][key].dtype


def test_writes_reference_checkpoint_format(tmp_path):
    mesh, graph = _small_graph()
    mesh.shutdown()
    params = vm.init_params(graph, 1)
    moments = {n: {k: np.full_like(v, 0.5) for k, v in b.items()} for n, b in params.items()}
    vm.save_checkpoint(tmp_path / "c", 7, params, moments, extra={"note": "x"})
    ref = json.loads(open(os.path.join(GOLD, "ref_checkpoint", "manifest.json")).read())
    got = json.loads((tmp_path / "c" / "manifest.json").read_text())
    assert got == ref
    for name in ref["blobs"]:
        a = np.load(tmp_path / "c" / name)
        b = np.load(os.path.join(GOLD, "ref_checkpoint", name))
        assert a.dtype == b.dtype and np.array_equal(a, b)
    step, p2, m2 = vm.load_checkpoint(tmp_path / "c")
    assert step == 7 and all(np.array_equal(p2[n]["kernel"], params[n]["kernel"]) for n in params)


@pytest.mark.parametrize("seed", [0, 11])
@pytest.mark.parametrize("bs", [1, 2])
def test_batch_order_matches_reference(seed, bs):
    gold = np.load(os.path.join(GOLD, "training_golden.npz"))[f"order_seed{seed}_bs{bs}"]
    recs = [(np.full((2, 2, 2), float(i), np.float32), np.zeros((2, 2, 2), np.uint8)) for i in range(5)]
    src = vm.BatchSource(recs, bs, seed)
    order = [[int(img[j, 0, 0, 0, 0]) for j in range(bs)] for img, _ in (src.batch(s) for s in range(12))]
    assert np.array_equal(np.array(order), gold)
    img, lab = src.batch(3)
    assert img.shape == (bs, 2, 2, 2, 1) and img.dtype == np.float32 and lab.dtype == np.uint8


def test_dice_known_answers():
    a = np.zeros((4, 4, 4), np.uint8)
    b = np.full((4, 4, 4), 2, np.uint8)
    assert vm.dice_per_case([b.copy(), b.copy()], [b.copy(), b.copy()]) == 1.0
    assert vm.dice_per_case([b, a], [b, b]) == pytest.approx(0.5)
    with pytest.raises(VoxmeshError):
        vm.dice_per_case([a], [a, b])
    a_pred = np.zeros(100, np.uint8)
    a_gt = np.zeros(100, np.uint8)
    a_pred[:10] = 2
    a_gt[10:20] = 2
    c = np.zeros(100, np.uint8)
    c[:90] = 2
    assert vm.dice_per_case([a_pred, c], [a_gt, c]) == pytest.approx(0.5)
    assert vm.dice_global([a_pred, c], [a_gt, c]) == pytest.approx(0.9)
    assert vm.dice_global([a_pred], [a_gt]) == 0.0
    empty = np.zeros((3, 3, 3), np.uint8)
    full = np.full((3, 3, 3), 2, np.uint8)
    assert vm.hard_dice(empty == 2, empty == 2) == 1.0
    assert vm.hard_dice(full == 2, empty == 2) == 0.0
    assert vm.dice_global([empty], [empty]) == 1.0


def test_dice_per_case_brute_force():
    rng = np.random.default_rng(3)
    preds = [rng.integers(0, 3, (5, 5, 5)).astype(np.uint8) for _ in range(6)]
    gts = [rng.integers(0, 3, (5, 5, 5)).astype(np.uint8) for _ in range(6)]
    scores = []
    for p, g in zip(preds, gts):
        pm, gm = p == 2, g == 2
        tot = pm.sum() + gm.sum()
        scores.append(1.0 if tot == 0 else 2 * np.logical_and(pm, gm).sum() / tot)
    assert vm.dice_per_case(preds, gts) == pytest.approx(float(np.mean(scores)), rel=1e-12)


def test_train_loop_rejects_augmentation():
    mesh, graph = _small_graph()
    mesh.shutdown()
    with pytest.raises(VoxmeshError):
        vm.train_loop(graph, [(np.zeros((8, 8, 8), np.float32), np.zeros((8, 8, 8), np.uint8))],
                      vm.TrainConfig(steps=1, augment=object()))
