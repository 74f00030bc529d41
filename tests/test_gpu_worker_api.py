"""The reference's worker-level hooks on the GPU step: unet.run_forward_local /
run_backward_local (unet.py:331-442), training.loss_stats_local / losses_from_stats /
loss_grad_local (training.py:77-127) and training.sgd_momentum_step (training.py:202-219),
driven exactly like the reference's _train_step (training.py:330-343), against the f64 oracle;
the distributed loss API (soft_dice_loss / cross_entropy_loss / combined_loss) on the loss
kernels against the reference's known answers (test_training.py:58-86)."""

import numpy as np
import pytest
import torch

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200 import training as T
from paper_1909_03108_b200 import unet as U
from tests.helpers import node_tuples, rel_l2

pytestmark = pytest.mark.gpu


def _train_step(ctx, graph, params, x, oh, total):
    """training._train_step (training.py:330-343) through the worker hooks."""
    probs, tape = U.run_forward_local(ctx, graph, params, x)
    stats = ctx.all_reduce_sum(T.loss_stats_local(probs, oh), tag="loss-stats")
    rc = T._RunCtx(3, (1, 2), 0.9, 0.1, 1e-12, total)
    dprobs = T.loss_grad_local(probs, oh, stats, rc)
    grads = U.run_backward_local(ctx, graph, params, tape, dprobs)
    return probs.cpu().numpy(), T.losses_from_stats(stats, rc), grads


@pytest.mark.parametrize("axes,layout", [([("one", 1)], {}), ([("mx", 2)], {"x": "mx"})])
def test_worker_hooks_fp32_match_f64_oracle(axes, layout):
    E = 16
    cfg = vm.UNetConfig(E, (8, 16), convs_per_block=2)
    img, lab = O.record_for(E, 0)
    x = img[None, ..., None].astype(np.float32)
    oh = O.one_hot(lab[None], 3).astype(np.float32)
    with vm.create_mesh(axes, backend="threads") as mesh:
        graph = vm.build(cfg, mesh, layout)
        params = vm.init_params(graph, 1)
        from paper_1909_03108_b200.training import _blocks

        xb = [torch.from_numpy(b).cuda() for b in _blocks(graph, x)]
        ob = [torch.from_numpy(b).cuda() for b in _blocks(graph, oh)]
        res = mesh.run(lambda ctx, xx, oo: _train_step(ctx, graph, params, xx, oo, E ** 3), per_worker=(xb, ob))
    with vm.create_mesh([("one", 1)]) as m1:
        g1 = vm.build(cfg, m1, {})
    p64 = {k: {kk: np.asarray(vv, np.float64) for kk, vv in v.items()} for k, v in params.items()}
    nodes = node_tuples(g1)
    rprobs, tape, _ = O.oracle_forward(nodes, p64, x.astype(np.float64))
    rstats = O.loss_stats(rprobs, oh.astype(np.float64))
    rloss = O.losses_from_stats(rstats, 3, E ** 3)
    rgrads, _ = O.oracle_backward(nodes, p64, tape, O.loss_grad(rprobs, oh.astype(np.float64), rstats, E ** 3))
    for (probs, loss, grads), rb in zip(res, _blocks(graph, rprobs)):
        assert rel_l2(probs, rb) <= 1e-5
        assert abs(loss[0] - rloss[0]) <= 1e-5 * abs(rloss[0])
        for k in rgrads:
            assert rel_l2(grads[k][0], rgrads[k][0]) <= 1e-5, k
            assert rel_l2(grads[k][1], rgrads[k][1]) <= 1e-5, k
    with pytest.raises(vm.VoxmeshError):  # the tape is consumed once
        tp = U.StepTape(None)
        tp.take()
        tp.take()


def test_sgd_momentum_step_is_numpys():
    rng = np.random.default_rng(4)
    params = {n: {"kernel": rng.standard_normal((3, 3, 3, 2, 4)).astype(np.float32),
                  "bias": rng.standard_normal(4).astype(np.float32)} for n in ("a", "b", "c")}
    moments = {n: {k: rng.standard_normal(v.shape).astype(np.float32) for k, v in b.items()} for n, b in params.items()}
    grads = {n: (rng.standard_normal((3, 3, 3, 2, 4)).astype(np.float32), rng.standard_normal(4).astype(np.float32))
             for n in params}
    grads["b"][0][0, 0, 0, 0, 0] = np.nan  # a non-finite layer is skipped (training.py:210-213)
    rp = {n: {k: v.copy() for k, v in b.items()} for n, b in params.items()}
    rm = {n: {k: v.copy() for k, v in b.items()} for n, b in moments.items()}
    rskip = O.sgd_momentum_step(rp, rm, grads, 0.003, 0.9, ("a", "b", "c"))
    skip = T.sgd_momentum_step(params, moments, grads, 0.003, 0.9, ("a", "b", "c"))
    assert skip == rskip == ["b"]
    for n in params:
        for k in ("kernel", "bias"):
            assert np.array_equal(params[n][k], rp[n][k]) and np.array_equal(moments[n][k], rm[n][k])


def test_distributed_losses_known_answers():
    # reference test_training.py:58-86: CE of a uniform prediction is ln 3; Dice 0.5 / 0.75
    with vm.create_mesh([("mx", 2)], backend="threads") as mesh:
        lay = vm.Layout({"x": "mx"})
        spec = vm.TensorSpec((("batch", 1), ("x", 4), ("y", 2), ("z", 2), ("c", 3)), "f32")
        probs = np.full(spec.shape, 1.0 / 3, dtype=np.float32)
        labels = np.zeros(spec.shape[:-1], dtype=np.int64)
        labels[0, :2] = 1
        labels[0, 2:] = 2
        oh = O.one_hot(labels, 3)
        ps, ohs = vm.shard(probs, spec, lay, mesh), vm.shard(oh, spec, lay, mesh)
        assert abs(vm.cross_entropy_loss(ps, ohs) - np.log(3.0)) <= 1e-6
        p2 = oh.copy()
        p2[0, 0, 0, 0] = [0, 0, 1]  # one class-1 voxel predicted as class 2
        ps2 = vm.shard(p2, spec, lay, mesh)
        want = 1.0 - 0.5 * ((2 * 7 / 15) + (2 * 8 / 17))
        assert abs(vm.soft_dice_loss(ps2, ohs) - want) <= 1e-6
        w = vm.LossWeights(0.9, 0.1)
        comb = vm.combined_loss(w, ps2, ohs)
        ce = vm.cross_entropy_loss(ps2, ohs)
        assert abs(comb - (0.9 * want + 0.1 * ce)) <= 1e-6
