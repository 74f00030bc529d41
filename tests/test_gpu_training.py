"""train_loop / checkpoints / evaluate on the GPU step (reference test_training.py:210-300)."""

import csv

import numpy as np
import pytest

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O

pytestmark = pytest.mark.gpu


def _records(n, extent=32, seed=7):
    return [O.record_for(extent, i, seed) for i in range(n)]


def _graph(mesh, layout=None):
    return vm.build(vm.UNetConfig(32, (16, 32), convs_per_block=2), mesh, layout or {})


def test_checkpoint_resume_is_bitwise(tmp_path):
    recs = _records(5)
    with vm.create_mesh([("one", 1)]) as mesh:
        full = vm.train_loop(_graph(mesh), recs, vm.TrainConfig(steps=6, lr=0.05, seed=11, log_every=0))
    with vm.create_mesh([("one", 1)]) as mesh:
        part = vm.train_loop(_graph(mesh), recs, vm.TrainConfig(steps=4, lr=0.05, seed=11, log_every=0))
        vm.save_checkpoint(tmp_path / "ck", part.step, part.params, part.moments)
    with vm.create_mesh([("one", 1)]) as mesh:
        resumed = vm.train_loop(_graph(mesh), recs, vm.TrainConfig(steps=2, lr=0.05, seed=11, log_every=0),
                                resume_from=tmp_path / "ck")
    assert resumed.step == full.step == 6
    for nid in full.params:
        for key in ("kernel", "bias"):
            assert np.array_equal(resumed.params[nid][key], full.params[nid][key]), (nid, key)
            assert np.array_equal(resumed.moments[nid][key], full.moments[nid][key]), (nid, key)
    assert [h[1] for h in resumed.history] == [h[1] for h in full.history[4:]]


def test_training_loss_decreases_and_writes_reference_files(tmp_path):
    recs = _records(3)
    cfg = vm.TrainConfig(steps=30, lr=0.05, seed=3, log_every=0, checkpoint_every=10, out_dir=str(tmp_path))
    with vm.create_mesh([("one", 1)]) as mesh:
        st = vm.train_loop(_graph(mesh), recs, cfg)
    losses = [h[1] for h in st.history]
    assert np.mean(losses[-5:]) < np.mean(losses[:5])
    rows = list(csv.reader(open(tmp_path / "metrics.csv")))
    assert rows[0] == ["step", "loss", "dice_loss", "ce_loss", "lr", "wall_ms"] and len(rows) == 31
    assert (tmp_path / "run.json").exists()
    for k in (10, 20, 30):
        step, p, m = vm.load_checkpoint(tmp_path / "checkpoints" / f"step_{k:06d}")
        assert step == k and set(p) == set(st.params)


def test_evaluate_reports_dice_and_loss():
    recs = _records(2)
    with vm.create_mesh([("one", 1)]) as mesh:
        g = _graph(mesh)
        vm.train_loop(g, recs, vm.TrainConfig(steps=3, lr=0.05, seed=1, log_every=0))
        out = vm.evaluate(g, recs, vm.TrainConfig())
    assert out["n_cases"] == 2
    assert 0.0 <= out["dice_per_case"] <= 1.0 and 0.0 <= out["dice_global"] <= 1.0
    assert np.isfinite(out["mean_loss"]) and out["mean_loss"] > 0


def test_two_rank_train_loop_tracks_single_rank():
    recs = _records(2)
    cfg = vm.TrainConfig(steps=3, lr=0.05, seed=5, log_every=0)
    with vm.create_mesh([("one", 1)]) as mesh:
        a = vm.train_loop(_graph(mesh), recs, cfg)
    with vm.create_mesh([("mx", 2)], backend="threads") as mesh:
        b = vm.train_loop(_graph(mesh, {"x": "mx"}), recs, cfg)
    la, lb = [h[1] for h in a.history], [h[1] for h in b.history]
    assert np.allclose(la, lb, rtol=1e-4), (la, lb)
