"""Parity at the configurations BASELINE.json names (VERDICT r01 "next round" item 1).

* cfg1 exactly: one halo-exchanging conv3d, 3x3x3, 16->16, 32^3 volume, 2-way depth split,
  fp32, through the reference's op API (``conv3d_forward`` / ``conv3d_backward``,
  ops.py:251-285) on a threads mesh: outputs and all three gradients <= 1e-5 rel-L2 against
  the f64 oracle, the halo-exchanged slabs bitwise the oracle's protocol (halo.py:109-155).
* cfg2 as benchmarked: the full 128^3 train step (recipe_for_resolution(128, 1/8), bench
  inputs: record 0 of dataset seed 7, init_params(seed 1)) against the REFERENCE's own f64
  dense network (tests/golden/cfg2_golden.npz, made by tests/golden/make_cfg2_golden.py):
  probabilities and loss <= 1e-2; every weight gradient's norm and the full gradients of
  five layers informational at <= 1e-1 (bf16 storage bound); then the
  per-op gate: each conv's forward, data gradient and weight gradient <= 1e-2 against the
  f64 oracle run on the step's own bf16 operands (teacher forcing).
* spatial partitions of the cfg4 ladder (recipe_for_resolution(512, 1.0) = 32..1024, six
  blocks) at a reduced 64^3 extent: a 2x2x2 mesh and the cfg5 layout b x mx x my (global
  batch 2) on the threads mesh, against the unpartitioned step on one rank and the f64
  oracle.
"""

import os

import numpy as np
import pytest
import torch

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200.step import UNetStep
from tests.helpers import node_tuples, rel_l2

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# ----------------------------------------------------------------------------- cfg1
def test_cfg1_single_conv_depth_split_fp32():
    E, C = 32, 16
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, E, E, E, C)).astype(np.float32)
    k = (rng.uniform(-1, 1, (3, 3, 3, C, C)) / np.sqrt(27 * C)).astype(np.float32)
    b = (0.1 * rng.standard_normal(C)).astype(np.float32)
    g = rng.standard_normal((1, E, E, E, C)).astype(np.float32)
    axes, lay = [("mx", 2)], {"x": "mx"}
    spec = vm.TensorSpec((("batch", 1), ("x", E), ("y", E), ("z", E), ("c", C)), "f32")
    with vm.create_mesh(axes, backend="threads") as mesh:
        layout = vm.Layout(lay)
        xs = vm.shard(x, spec, layout, mesh)
        padded = vm.halo_exchange(xs, vm.HaloSpec.for_kernel(3))
        mesh.synchronize()
        slabs = [p.data.cpu().numpy() for p in padded]
        y, tape = vm.conv3d_forward(xs, vm.ConvParams(k, b))
        gx, gk, gb = vm.conv3d_backward(vm.shard(g, spec, layout, mesh), tape)
        yg, gxg = vm.gather(y), vm.gather(gx)
    ref_slabs, nbytes = O.halo_exchange_blocks(O.shard_blocks(x, spec.dims, lay, axes), spec.dims, lay, axes,
                                                {d: (1, 1) for d in "xyz"})
    for got, ref in zip(slabs, ref_slabs):
        assert np.array_equal(got, ref)  # halo-exchanged slabs: bit-exact
    assert nbytes == 2 * 32 * 32 * 16 * 4  # one 64 KB face each way
    x64, k64, b64, g64 = (a.astype(np.float64) for a in (x, k, b, g))
    ry = O.conv3d_dense(x64, k64, b64)
    rgx, rgk, rgb = O.conv3d_dense_backward(g64, x64, k64)
    assert rel_l2(yg, ry) <= 1e-5
    assert rel_l2(gxg, rgx) <= 1e-5
    assert rel_l2(gk, rgk) <= 1e-5 and rel_l2(gb, rgb) <= 1e-5


# ----------------------------------------------------------------------------- cfg2
def _slab_dense(slab):
    return slab.interior().cpu().numpy().astype(np.float64)


def test_cfg2_full_step_against_reference_f64():
    gold = np.load(os.path.join(GOLD, "cfg2_golden.npz"))
    E = 128
    cfg = vm.recipe_for_resolution(E, 0.125)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 1)
    assert abs(sum(float(np.abs(v["kernel"]).sum()) for v in params.values()) - gold["param_sum"][0]) <= 1e-6 * \
        gold["param_sum"][0]
    from paper_1909_03108_b200.data import synth_record

    img, lab = synth_record(E, 7, 0)
    st = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
    st.keep_probs = True
    st.upload(torch.from_numpy(img[None, ..., None].copy()), torch.from_numpy(lab[None].copy()))
    st.forward()
    st.backward()
    torch.cuda.synchronize()
    probs = st.probs.reshape(-1, 3).cpu().numpy()[gold["probs_idx"]]
    assert rel_l2(probs, gold["probs"]) <= 1e-2
    assert rel_l2(st.stats.cpu().numpy(), gold["loss_stats"]) <= 1e-2
    loss = st.loss()
    assert abs(loss[0] - gold["loss_values"][0]) <= 1e-2 * abs(gold["loss_values"][0])
    grads = st.grad_dict()
    for nid, (gk, gb) in grads.items():  # end to end: storage-bound (informational tolerance)
        n = gold[f"gnorm_{nid}"]
        assert abs(np.linalg.norm(gk) - n[0]) <= 1e-1 * n[0], nid
        if f"gk_{nid}" in gold:
            assert rel_l2(gk, gold[f"gk_{nid}"]) <= 1e-1, nid
            assert rel_l2(gb, gold[f"gb_{nid}"]) <= 1e-1, nid

    # per-op gate (teacher forcing): the step's own bf16 operands through the f64 oracle
    nodes = {n.id: n for n in graph.nodes}
    for nid in ("enc0_conv1", "dec0_conv0", "enc1_conv1", "dec1_conv0", "enc3_conv2", "dec2_conv0"):
        L = st.by_id[nid]
        n = nodes[nid]
        x = _slab_dense(st.out[n.inputs[0]])
        gy = _slab_dense(st.gpre[nid])
        w = O.bf16_round(params[nid]["kernel"]).astype(np.float64)
        bias = params[nid]["bias"].astype(np.float64)
        y_ref = np.maximum(O.conv3d_dense(x, w, bias), 0)
        assert rel_l2(_slab_dense(st.out[nid]), y_ref) <= 1e-2, nid
        gx_ref, gk_ref, gb_ref = O.conv3d_dense_backward(gy, x, w)
        gk, gb = grads[nid]
        assert rel_l2(gk, gk_ref) <= 1e-2, nid
        assert rel_l2(gb, gb_ref) <= 1e-2, nid
        src = nodes[n.inputs[0]]
        if src.op == "relu":  # dgrad epilogue applies the producer's ReLU mask
            mask = _slab_dense(st.out[src.id]) > 0
            assert rel_l2(_slab_dense(st.gpre[src.inputs[0]]), np.where(mask, gx_ref, 0)) <= 1e-2, nid
    mesh.shutdown()


# ----------------------------------------------------------------------------- cfg4 / cfg5 ladders
def _cfg4_small(E=64):
    full = vm.recipe_for_resolution(512, 1.0)
    return vm.UNetConfig(E, full.encoder_filters, convs_per_block=full.convs_per_block)


def _run_partitioned(cfg, params, axes, layout, img, lab):
    """Every rank's step on the threads mesh (one GPU); returns per-rank (loss, grads, probs)."""
    mesh = vm.create_mesh(axes, backend="threads")
    g = vm.build(cfg, mesh, layout)
    from paper_1909_03108_b200.training import _blocks

    E = cfg.input_extent
    bi = [torch.from_numpy(b) for b in _blocks(g, img)]
    bl = [torch.from_numpy(b) for b in _blocks(g, lab)]
    bdim = layout.get("batch")
    B = img.shape[0] // (mesh.axis_size(bdim) if bdim else 1)

    def work(ctx, im, lb):
        st = UNetStep(g, params, batch=B, ctx=ctx, dtype=torch.bfloat16, global_shape=(E, E, E),
                      global_batch=img.shape[0])
        st.keep_probs = True
        st.upload(im, lb)
        st.forward()
        st.backward()
        st.all_reduce_grads()
        torch.cuda.synchronize()
        return st.loss()[0], st.grad_dict(), st.probs.reshape(tuple(im.shape[:4]) + (-1,)).cpu().numpy()

    res = mesh.run(work, per_worker=(bi, bl))
    mesh.shutdown()
    return g, res


@pytest.mark.parametrize("axes,layout,batch", [
    ([("mx", 2), ("my", 2), ("mz", 2)], {"x": "mx", "y": "my", "z": "mz"}, 1),   # cfg4's 2x2x2 mesh
    ([("b", 2), ("mx", 2), ("my", 2)], {"batch": "b", "x": "mx", "y": "my"}, 2),  # cfg5's layout
])
def test_cfg4_ladder_partitioned_matches_single_rank_and_oracle(axes, layout, batch):
    E = 64
    cfg = _cfg4_small(E)
    m1 = vm.create_mesh([("one", 1)])
    g1 = vm.build(cfg, m1, {})
    params = vm.init_params(g1, 2)
    recs = [O.record_for(E, i) for i in range(batch)]
    img = np.stack([r[0] for r in recs])[..., None].astype(np.float32)
    lab = np.stack([r[1] for r in recs]).astype(np.uint8)
    st = UNetStep(g1, params, batch=batch, dtype=torch.bfloat16, device="cuda")
    st.keep_probs = True
    st.upload(torch.from_numpy(img), torch.from_numpy(lab))
    st.forward()
    st.backward()
    torch.cuda.synchronize()
    loss1, grads1 = st.loss()[0], st.grad_dict()
    probs1 = st.probs.reshape(batch, E, E, E, 3).cpu().numpy()
    m1.shutdown()

    g, res = _run_partitioned(cfg, params, axes, layout, img, lab)
    from paper_1909_03108_b200.training import _blocks

    # the conv planners pick per block shape (64^3 vs 32^3 blocks: different accumulator
    # splits), so bf16 roundings differ between the two runs: bf16 tolerances, and both
    # against the f64 oracle below
    ref_blocks = _blocks(g, probs1)
    for (loss, grads, probs), rb in zip(res, ref_blocks):
        assert abs(loss - loss1) <= 1e-3 * abs(loss1)
        assert rel_l2(probs, rb) <= 1e-2
    for _, grads, _ in res[1:]:  # every rank holds the same all-reduced gradient, bitwise
        for k in grads:
            assert np.array_equal(grads[k][0], res[0][1][k][0])

    # against the f64 oracle (SURVEY §8(c) protocol): probabilities and loss <= 1e-2; the
    # end-to-end bf16 weight gradients are storage-bound (the 2^3-voxel bottleneck of this
    # reduced ladder reaches ~0.2 on ONE rank too, tools/dbg_cfg4_ladder.py), so the gate is
    # that partitioning does not move them further from f64 than the single rank is
    oh = O.one_hot(lab, 3).astype(np.float64)
    p64 = {k: {kk: np.asarray(vv, np.float64) for kk, vv in v.items()} for k, v in params.items()}
    nodes = node_tuples(g1)
    rprobs, tape, _ = O.oracle_forward(nodes, p64, img.astype(np.float64))
    assert rel_l2(probs1, rprobs) <= 1e-2
    for (_, _, probs), rb in zip(res, _blocks(g, rprobs)):
        assert rel_l2(probs, rb) <= 1e-2
    total = int(np.prod(img.shape[:4]))
    rstats = O.loss_stats(rprobs, oh)
    rloss = O.losses_from_stats(rstats, 3, total)[0]
    assert abs(loss1 - rloss) <= 1e-2 * abs(rloss)
    rgrads, _ = O.oracle_backward(nodes, p64, tape, O.loss_grad(rprobs, oh, rstats, total))
    for k, (gk, _) in rgrads.items():
        e1, ep = rel_l2(grads1[k][0], gk), rel_l2(res[0][1][k][0], gk)
        assert ep <= 1.25 * e1 + 2e-2, (k, ep, e1)


# ----------------------------------------------------------------------------- evaluation
def test_eval_argmax_and_dice_counts_are_exact():
    E = 32
    cfg = vm.UNetConfig(E, (16, 32), convs_per_block=1)
    mesh = vm.create_mesh([("one", 1)])
    g = vm.build(cfg, mesh, {})
    params = vm.init_params(g, 3)
    img, lab = O.record_for(E, 2)
    st = UNetStep(g, params, dtype=torch.bfloat16, device="cuda")
    st.keep_probs, st.keep_pred = True, True
    st.upload(torch.from_numpy(img[None, ..., None].copy()), torch.from_numpy(lab[None].copy()))
    st.forward()
    from paper_1909_03108_b200 import _lib

    counts = torch.zeros(9, dtype=torch.int64, device="cuda")
    _lib.call("vm_label_counts", _lib.ptr(st.pred), _lib.ptr(st.labels), st.nvox, 3, _lib.ptr(counts),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    probs = st.probs.reshape(-1, 3).cpu().numpy()
    pred = st.pred.cpu().numpy()
    assert np.array_equal(pred, np.argmax(probs, axis=-1).astype(np.uint8))  # np.argmax semantics
    gt = lab.reshape(-1)
    want = [int(np.count_nonzero((pred == k) & (gt == k))) for k in range(3)]
    want += [int(np.count_nonzero(pred == k)) for k in range(3)] + [int(np.count_nonzero(gt == k)) for k in range(3)]
    assert counts.cpu().numpy().tolist() == want
    mesh.shutdown()


def test_evaluate_matches_oracle_pipeline_and_layouts():
    E = 32
    cfg = vm.UNetConfig(E, (16, 32), convs_per_block=1)
    recs = [O.record_for(E, i) for i in range(3)]
    with vm.create_mesh([("one", 1)]) as mesh:
        g = vm.build(cfg, mesh, {})
        params = vm.init_params(g, 4)
        out1 = vm.evaluate(g, recs, vm.TrainConfig(), params=params)
    # the oracle pipeline: f64 forward -> argmax -> hard Dice of the tumour class; per-sample loss
    nodes = node_tuples(g)
    p64 = {k: {kk: np.asarray(vv, np.float64) for kk, vv in v.items()} for k, v in params.items()}
    preds, losses = [], []
    for im, lb in recs:
        pr, _, _ = O.oracle_forward(nodes, p64, im[None, ..., None].astype(np.float64))
        preds.append(np.argmax(pr[0], axis=-1))
        losses.append(O.losses_from_stats(O.loss_stats(pr, O.one_hot(lb[None], 3).astype(np.float64)), 3,
                                          E ** 3)[0])
    gts = [r[1] for r in recs]
    assert abs(out1["dice_per_case"] - vm.dice_per_case(preds, gts)) <= 2e-2
    assert abs(out1["dice_global"] - vm.dice_global(preds, gts)) <= 2e-2
    assert abs(out1["mean_loss"] - np.mean(losses)) <= 1e-2 * np.mean(losses)
    # a data-parallel x spatial layout with a padded last chunk gives the same numbers
    with vm.create_mesh([("b", 2), ("mx", 2)], backend="threads") as mesh:
        g2 = vm.build(cfg, mesh, {"batch": "b", "x": "mx"})
        out2 = vm.evaluate(g2, recs, vm.TrainConfig(), params=params)
    assert out2["n_cases"] == 3
    for key in ("dice_per_case", "dice_global"):  # kernels may differ per block shape: argmax near-ties
        assert abs(out2[key] - out1[key]) <= 2e-2, key
    assert abs(out2["mean_loss"] - out1["mean_loss"]) <= 1e-3 * out1["mean_loss"]
