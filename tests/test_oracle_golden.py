"""The CPU oracle port vs golden vectors produced by the reference itself (tests/golden/)."""

import os

import numpy as np
import pytest

from oracle import voxmesh_oracle as O

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "voxmesh_golden.npz"))
AXES = [("mx", 2), ("my", 2), ("mz", 2)]
LAY = {"x": "mx", "y": "my", "z": "mz"}
DIMS = (("batch", 1), ("x", 8), ("y", 8), ("z", 8), ("c", 2))


def test_halo_forward_bitwise_and_bytes():
    x = G["halo_x"]
    padded, nbytes = O.halo_exchange_blocks(O.shard_blocks(x, DIMS, LAY, AXES), DIMS, LAY, AXES,
                                            {d: (1, 1) for d in "xyz"})
    for r in range(8):
        assert np.array_equal(padded[r], G[f"halo_padded_{r}"])
    assert nbytes == int(G["halo_bytes"])
    assert O.exchange_byte_count(DIMS, LAY, AXES, {d: (1, 1) for d in "xyz"}, 4) == int(G["halo_bytes"])


def test_halo_adjoint_bitwise():
    ys = [G[f"halo_bwd_in_{r}"] for r in range(8)]
    out = O.halo_exchange_backward_blocks(ys, DIMS, LAY, AXES, {d: (1, 1) for d in "xyz"})
    assert np.array_equal(O.gather_blocks(out, DIMS, LAY, AXES, np.float32), G["halo_bwd_out"])


def test_halo_asymmetric_margins_bitwise():
    dims = (("x", 8), ("y", 4))
    padded, _ = O.halo_exchange_blocks(O.shard_blocks(G["asym_x"], dims, {"x": "mx"}, [("mx", 2)]), dims,
                                       {"x": "mx"}, [("mx", 2)], {"x": (2, 1), "y": (1, 2)})
    assert np.array_equal(padded[0], G["asym_padded_0"])
    assert np.array_equal(padded[1], G["asym_padded_1"])


def test_halo_1d_hand_checked():
    # test_halo.py:54-64 and :163-171 known answers
    dims = (("x", 8),)
    padded, _ = O.halo_exchange_blocks(O.shard_blocks(np.arange(8, dtype=np.float32), dims, {"x": "ax"}, [("ax", 2)]),
                                       dims, {"x": "ax"}, [("ax", 2)], {"x": (1, 1)})
    assert padded[0].tolist() == [0, 0, 1, 2, 3, 4] and padded[1].tolist() == [3, 4, 5, 6, 7, 0]
    back = O.halo_exchange_backward_blocks([np.ones(6, np.float32)] * 2, dims, {"x": "ax"}, [("ax", 2)], {"x": (1, 1)})
    assert back[0].tolist() == [1, 1, 1, 2] and back[1].tolist() == [2, 1, 1, 1]


def test_byte_counts_of_baseline_configs():
    cases = [
        (256, [("mx", 2)], {"x": "mx"}),
        (256, [("mx", 4)], {"x": "mx"}),
        (256, [("mx", 8)], {"x": "mx"}),
        (512, AXES, LAY),
        (512, [("b", 2), ("mx", 2), ("my", 2)], {"batch": "b", "x": "mx", "y": "my"}),
    ]
    for (ext, ax, lo), want in zip(cases, G["byte_counts_c32_f32"]):
        b = 2 if "batch" in lo else 1
        dims = (("batch", b), ("x", ext), ("y", ext), ("z", ext), ("c", 32))
        assert O.exchange_byte_count(dims, lo, ax, {d: (1, 1) for d in "xyz"}, 4) == int(want)


@pytest.mark.parametrize("dt,tol", [("f32", 2e-6), ("f64", 1e-13)])
def test_dense_conv_matches_reference(dt, tol):
    y = O.conv3d_dense(G[f"conv_{dt}_x"], G[f"conv_{dt}_k"], G[f"conv_{dt}_b"])
    assert O.rel_l2(y, G[f"conv_{dt}_y"]) <= tol
    gx, gk, gb = O.conv3d_dense_backward(G[f"conv_{dt}_gout"], G[f"conv_{dt}_x"], G[f"conv_{dt}_k"])
    for got, key in ((gx, "gx"), (gk, "gk"), (gb, "gb")):
        assert O.rel_l2(got, G[f"conv_{dt}_{key}"]) <= tol


def test_pool_upsample_softmax_bitwise():
    y, idx = O.maxpool2_dense(G["pool_x"])
    assert np.array_equal(y, G["pool_y"]) and np.array_equal(idx, G["pool_idx"])
    assert np.array_equal(O.maxpool2_dense_backward(G["pool_gout"], idx, G["pool_x"].shape), G["pool_gin"])
    assert np.array_equal(O.upsample2_dense(G["up_x"]), G["up_y"])
    assert np.array_equal(O.upsample2_dense_backward(G["up_gout"]), G["up_gin"])
    assert np.array_equal(O.softmax_dense(G["sm_x"]), G["sm_p"])
    assert np.array_equal(O.softmax_dense_backward(G["sm_gout"], G["sm_p"]), G["sm_gin"])


def test_loss_stats_value_and_gradient():
    oh = O.one_hot(G["loss_labels"], 3)
    st = O.loss_stats(G["loss_probs"], oh)
    assert np.array_equal(st, G["loss_stats"])
    vals = O.losses_from_stats(st, 3, 2 * 4 ** 3)
    assert np.allclose(vals, G["loss_values"], rtol=0, atol=0)
    assert np.array_equal(O.loss_grad(G["loss_probs"], oh, st, 2 * 4 ** 3), G["loss_grad"])


def test_sgd_step_bitwise_and_nonfinite_skip():
    params = {k: {kk: G[f"sgd_p0_{k}_{kk}"].copy() for kk in ("kernel", "bias")} for k in "ab"}
    moms = {k: {kk: G[f"sgd_v0_{k}_{kk}"].copy() for kk in ("kernel", "bias")} for k in "ab"}
    grads = {k: (G[f"sgd_g_{k}_kernel"], G[f"sgd_g_{k}_bias"]) for k in "ab"}
    skipped = O.sgd_momentum_step(params, moms, grads, 0.003, 0.9, ("a", "b"))
    assert skipped == list(G["sgd_skipped"])
    for k in "ab":
        for kk in ("kernel", "bias"):
            assert np.array_equal(params[k][kk], G[f"sgd_p1_{k}_{kk}"])
            assert np.array_equal(moms[k][kk], G[f"sgd_v1_{k}_{kk}"])


def test_recipes_graph_and_init():
    for row in G["recipes"]:
        ext, sc = int(row[0]), float(row[1])
        want = tuple(int(v) for v in row[2:] if v)
        assert O.recipe_filters(ext, sc) == want
    for name, (ext, sc) in (("cfg2", (128, 0.125)), ("cfg4", (512, 1.0))):
        nodes = O.graph_nodes(O.recipe_filters(ext, sc))
        assert [n[0] for n in nodes] == list(G[f"graph_{name}_ids"])
        assert [n[1] for n in nodes] == list(G[f"graph_{name}_ops"])
        assert [n[4] for n in nodes] == list(G[f"graph_{name}_cin"])
    nodes = O.graph_nodes((2, 4), convs_per_block=2)
    params = O.init_params(nodes, 5)
    for nid, d in params.items():
        assert np.array_equal(d["kernel"], G[f"net_p_{nid}_kernel"])


def test_dense_network_forward_backward_f64():
    nodes = O.graph_nodes((2, 4), convs_per_block=2)
    p = {k: {kk: vv.astype(np.float64) for kk, vv in v.items()} for k, v in O.init_params(nodes, 5).items()}
    x = G["net_x"].astype(np.float64)
    oh = O.one_hot(G["net_labels"], 3, np.float64)
    probs, tape, _ = O.oracle_forward(nodes, p, x)
    assert O.rel_l2(probs, G["net_probs_f64"]) <= 1e-13
    st = O.loss_stats(probs, oh)
    grads, _ = O.oracle_backward(nodes, p, tape, O.loss_grad(probs, oh, st, 8 ** 3))
    for nid, (gk, gb) in grads.items():
        assert O.rel_l2(gk, G[f"net_gk_{nid}"]) <= 1e-12
        assert O.rel_l2(gb, G[f"net_gb_{nid}"]) <= 1e-12


def test_synthetic_record_bitwise():
    img, lab = O.record_for(16, 0)
    assert np.array_equal(img, G["synth16_image"]) and np.array_equal(lab, G["synth16_labels"])


def test_loss_closed_forms():
    # test_training.py:58-86: CE of uniform = ln 3; all-tumour dice 0.5 / 0.75; combined 0.55986
    oh = O.one_hot(np.full((1, 4, 4, 4), 2, np.uint8), 3)
    probs = np.full_like(oh, 1 / 3)
    st = O.loss_stats(probs, oh)
    comb, dice, ce = O.losses_from_stats(st, 3, 64, dice_classes=(2,))
    assert abs(ce - np.log(3)) <= 1e-6 and abs(dice - 0.5) <= 1e-6 and abs(comb - 0.55986) <= 1e-4
    assert abs(O.losses_from_stats(st, 3, 64)[1] - 0.75) <= 1e-6
