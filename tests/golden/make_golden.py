"""Generate tests/golden/voxmesh_golden.npz by running the REFERENCE implementation.

Run in the build container, where the read-only reference lives:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``voxmesh`` from /root/reference/pkg/src and records inputs/outputs of the
hot-path functions (halo exchange fwd/adjoint + byte counts, dense conv fwd/bwd,
pool/upsample/softmax, loss statistics and gradient, SGD, U-Net builder, init,
dense network fwd/bwd, synthetic record).  The GPU box never reads /root/reference:
tests compare the oracle port and the CUDA path against these committed vectors.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "voxmesh_golden.npz")


def main():
    sys.path.insert(0, REF)
    import voxmesh  # noqa: F401
    from voxmesh import halo, oracle, training, unet
    from voxmesh.data_io import synthesize_record
    from voxmesh.mesh import create_mesh
    from voxmesh.sharding import Layout, TensorSpec, gather, shard

    g = {}
    rng = np.random.default_rng(20260)

    # ---- halo on a 2x2x2 mesh (test_halo.py:81-93 shape), forward + adjoint
    axes = [("mx", 2), ("my", 2), ("mz", 2)]
    lay = {"x": "mx", "y": "my", "z": "mz"}
    spec = TensorSpec((("batch", 1), ("x", 8), ("y", 8), ("z", 8), ("c", 2)), "f32")
    x = rng.standard_normal(spec.shape).astype(np.float32)
    hs = halo.HaloSpec.for_kernel(3)
    with create_mesh(axes) as mesh:
        st = shard(x, spec, Layout(lay), mesh)
        b0 = mesh.run(lambda ctx: ctx.counters["p2p_bytes"])
        padded = halo.halo_exchange(st, hs)
        b1 = mesh.run(lambda ctx: ctx.counters["p2p_bytes"])
        g["halo_x"] = x
        for r, pb in enumerate(padded):
            g[f"halo_padded_{r}"] = pb.data
        g["halo_bytes"] = np.int64(sum(b1) - sum(b0))
        ys = [rng.standard_normal(pb.data.shape).astype(np.float32) for pb in padded]
        back = halo.halo_exchange_backward(ys, spec, Layout(lay), mesh, hs)
        for r, y in enumerate(ys):
            g[f"halo_bwd_in_{r}"] = y
        g["halo_bwd_out"] = gather(back)
    # asymmetric margins, partially sharded (test_halo.py:113-126)
    with create_mesh([("mx", 2)]) as mesh:
        spec2 = TensorSpec((("x", 8), ("y", 4)))
        h2 = halo.HaloSpec((("x", 2, 1), ("y", 1, 2)))
        x2 = rng.standard_normal(spec2.shape).astype(np.float32)
        padded = halo.halo_exchange(shard(x2, spec2, Layout({"x": "mx"}), mesh), h2)
        g["asym_x"] = x2
        g["asym_padded_0"] = padded[0].data
        g["asym_padded_1"] = padded[1].data
    # byte counts of the BASELINE configs at itemsize 4 (f32; scale for bf16)
    counts = []
    for ext, ax, lo in [
        (256, [("mx", 2)], {"x": "mx"}),
        (256, [("mx", 4)], {"x": "mx"}),
        (256, [("mx", 8)], {"x": "mx"}),
        (512, [("mx", 2), ("my", 2), ("mz", 2)], {"x": "mx", "y": "my", "z": "mz"}),
        (512, [("b", 2), ("mx", 2), ("my", 2)], {"batch": "b", "x": "mx", "y": "my"}),
    ]:
        with create_mesh([(n, 1) for n, _ in ax]) as _m:
            pass
        # exchange_byte_count needs only mesh metadata; a thin stand-in avoids 8 threads
        class _M:
            pass

        m = _M()
        m.axes = [type("A", (), {"name": n, "size": s})() for n, s in ax]
        m.axis_index = {n: i for i, (n, _) in enumerate(ax)}
        m.coords = [c for c in np.ndindex(*[s for _, s in ax])]
        m.axis_size = lambda a, _ax=dict(ax): _ax[a]
        batch = 2 if "batch" in lo else 1
        sp = TensorSpec((("batch", batch), ("x", ext), ("y", ext), ("z", ext), ("c", 32)), "f32")
        counts.append(halo.exchange_byte_count(sp, Layout(lo), m, hs))
    g["byte_counts_c32_f32"] = np.array(counts, dtype=np.int64)

    # ---- dense conv fwd / bwd (oracle.py:23-76), f32 and f64
    for dt in ("f32", "f64"):
        npdt = np.float32 if dt == "f32" else np.float64
        xc = rng.standard_normal((2, 6, 7, 5, 3)).astype(npdt)
        k = rng.standard_normal((3, 3, 3, 3, 4)).astype(npdt)
        bb = rng.standard_normal(4).astype(npdt)
        go = rng.standard_normal((2, 6, 7, 5, 4)).astype(npdt)
        g[f"conv_{dt}_x"], g[f"conv_{dt}_k"], g[f"conv_{dt}_b"], g[f"conv_{dt}_gout"] = xc, k, bb, go
        g[f"conv_{dt}_y"] = oracle.conv3d_dense(xc, k, bb)
        gx, gk, gb = oracle.conv3d_dense_backward(go, xc, k)
        g[f"conv_{dt}_gx"], g[f"conv_{dt}_gk"], g[f"conv_{dt}_gb"] = gx, gk, gb

    # ---- pool / upsample / softmax
    xp = rng.standard_normal((1, 4, 6, 8, 3)).astype(np.float32)
    xp[0, :2, :2, :2, 0] = 1.0  # a tie cell
    pooled, idx = oracle.maxpool2_dense(xp)
    gp = rng.standard_normal(pooled.shape).astype(np.float32)
    g["pool_x"], g["pool_y"], g["pool_idx"] = xp, pooled, idx
    g["pool_gout"], g["pool_gin"] = gp, oracle.maxpool2_dense_backward(gp, idx, xp.shape)
    xu = rng.standard_normal((1, 2, 3, 2, 4)).astype(np.float32)
    gu = rng.standard_normal((1, 4, 6, 4, 4)).astype(np.float32)
    g["up_x"], g["up_y"], g["up_gout"], g["up_gin"] = xu, oracle.upsample2_dense(xu), gu, oracle.upsample2_dense_backward(gu)
    xs = rng.standard_normal((2, 3, 3, 3, 3)).astype(np.float32)
    ps = oracle.softmax_dense(xs)
    gs = rng.standard_normal(xs.shape).astype(np.float32)
    g["sm_x"], g["sm_p"], g["sm_gout"], g["sm_gin"] = xs, ps, gs, oracle.softmax_dense_backward(gs, ps)

    # ---- loss statistics / value / gradient (training.py:77-127)
    labels = rng.integers(0, 3, (2, 4, 4, 4)).astype(np.uint8)
    oh = training.one_hot(labels, 3)
    logits = rng.standard_normal(oh.shape).astype(np.float32)
    probs = (np.exp(logits) / np.exp(logits).sum(-1, keepdims=True)).astype(np.float32)
    stats = training.loss_stats_local(probs, oh)
    rc = training._RunCtx(3, (1, 2), 0.9, 0.1, 1e-12, 2 * 4 ** 3, 0.003, 0.9, param_order=())
    g["loss_labels"], g["loss_probs"], g["loss_stats"] = labels, probs, stats
    g["loss_values"] = np.array(training.losses_from_stats(stats, rc), dtype=np.float64)
    g["loss_grad"] = training.loss_grad_local(probs, oh, stats, rc)

    # ---- SGD with momentum (training.py:202-219), incl. a non-finite layer
    params = {"a": {"kernel": rng.standard_normal((3, 3, 3, 2, 2)).astype(np.float32),
                    "bias": rng.standard_normal(2).astype(np.float32)},
              "b": {"kernel": rng.standard_normal((1, 1, 1, 2, 3)).astype(np.float32),
                    "bias": rng.standard_normal(3).astype(np.float32)}}
    moms = {k: {kk: rng.standard_normal(vv.shape).astype(np.float32) for kk, vv in v.items()} for k, v in params.items()}
    grads = {k: (rng.standard_normal(v["kernel"].shape).astype(np.float32), rng.standard_normal(v["bias"].shape).astype(np.float32))
             for k, v in params.items()}
    grads["b"][0][0, 0, 0, 0, 0] = np.inf
    for k in params:
        for kk in ("kernel", "bias"):
            g[f"sgd_p0_{k}_{kk}"] = params[k][kk].copy()
            g[f"sgd_v0_{k}_{kk}"] = moms[k][kk].copy()
        g[f"sgd_g_{k}_kernel"], g[f"sgd_g_{k}_bias"] = grads[k]
    skipped = training.sgd_momentum_step(params, moms, grads, 0.003, 0.9, ("a", "b"))
    for k in params:
        for kk in ("kernel", "bias"):
            g[f"sgd_p1_{k}_{kk}"] = params[k][kk]
            g[f"sgd_v1_{k}_{kk}"] = moms[k][kk]
    g["sgd_skipped"] = np.array(skipped)

    # ---- U-Net recipes / builder / init / dense network fwd+bwd
    recipes = []
    for ext, sc in [(16, 1.0), (32, 1.0), (64, 1.0), (128, 1.0), (128, 0.125), (256, 0.5), (512, 1.0)]:
        cfg = unet.recipe_for_resolution(ext, sc)
        recipes.append([ext, sc] + list(cfg.encoder_filters) + [0] * (8 - len(cfg.encoder_filters)))
    g["recipes"] = np.array(recipes, dtype=np.float64)
    with create_mesh([("one", 1)]) as mesh:
        for name, cfg in [("cfg2", unet.recipe_for_resolution(128, 0.125)), ("cfg4", unet.recipe_for_resolution(512, 1.0))]:
            graph = unet.build(cfg, mesh, Layout({}))
            g[f"graph_{name}_ids"] = np.array([n.id for n in graph.nodes])
            g[f"graph_{name}_ops"] = np.array([n.op for n in graph.nodes])
            g[f"graph_{name}_cin"] = np.array([n.c_in for n in graph.nodes])
            g[f"graph_{name}_cout"] = np.array([n.c_out for n in graph.nodes])
            g[f"graph_{name}_params"] = np.int64(graph.param_count)
            g[f"graph_{name}_rf"] = np.int64(graph.receptive_field())
        cfg = unet.UNetConfig(8, (2, 4), convs_per_block=2)
        graph = unet.build(cfg, mesh, Layout({}))
        p = unet.init_params(graph, 5)
        for nid, d in p.items():
            g[f"net_p_{nid}_kernel"] = d["kernel"]
        xn = rng.standard_normal((1, 8, 8, 8, 1)).astype(np.float32)
        ln = rng.integers(0, 3, (1, 8, 8, 8)).astype(np.uint8)
        ohn = training.one_hot(ln, 3)
        p64 = {k: {kk: vv.astype(np.float64) for kk, vv in v.items()} for k, v in p.items()}
        probs, tape = oracle.oracle_forward(graph, p64, xn.astype(np.float64))
        st64 = training.loss_stats_local(probs, ohn.astype(np.float64))
        rc = training._RunCtx(3, (1, 2), 0.9, 0.1, 1e-12, 8 ** 3, 0.0, 0.0, param_order=())
        d = training.loss_grad_local(probs, ohn.astype(np.float64), st64, rc)
        pg, _ = oracle.oracle_backward(graph, p64, tape, d)
        g["net_x"], g["net_labels"], g["net_probs_f64"] = xn, ln, probs
        for nid, (gk, gb) in pg.items():
            g[f"net_gk_{nid}"], g[f"net_gb_{nid}"] = gk, gb

    # ---- synthetic record (data_io.py:163-184), dataset seed 7, record 0
    rec = synthesize_record(16, np.random.default_rng(np.random.SeedSequence([7, 0])), "case000")
    g["synth16_image"], g["synth16_labels"] = rec.image, rec.labels

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
