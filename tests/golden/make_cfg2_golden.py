"""Generate tests/golden/cfg2_golden.npz: the REFERENCE's f64 dense network on the benchmarked
cfg2 workload (recipe_for_resolution(128, 1/8) = (16, 32, 64, 128), 128^3, batch 1).

Run in the build container, where the read-only reference lives (takes tens of minutes:
the reference convolution is single-threaded ``einsum(optimize=False)``):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cfg2_golden.py

Inputs are exactly the bench's: record 0 of dataset seed 7 (``data_io.synthesize_record``
with ``SeedSequence([7, 0])``, data_io.py:163-196) and ``unet.init_params(graph, 1)``
(unet.py:284-299).  The reference runs ``oracle.oracle_forward`` / ``oracle_backward``
(oracle.py:126-202) in float64 on those values, with ``training.loss_stats_local`` /
``losses_from_stats`` / ``loss_grad_local`` (training.py:77-127) in between.

Stored (the full 128^3 arrays are too large to commit):
* ``loss_stats`` (10), ``loss_values`` (combined, dice, ce);
* ``probs_idx`` / ``probs`` — the f64 class probabilities at 32768 seeded voxel indices;
* ``gk_<id>`` / ``gb_<id>`` (float32) for a few layers, ``gnorm_<id>`` (||gk||, ||gb||) for all;
* ``param_sum`` — a checksum of the init draws, so a drift in init is caught first.
The GPU box never reads /root/reference: tests/test_gpu_configs.py compares against this file.
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg2_golden.npz")
FULL_GRAD_LAYERS = ("enc0_conv0", "enc0_conv1", "dec0_conv0", "enc1_conv1", "head")


def main():
    sys.path.insert(0, REF)
    from voxmesh import oracle, training, unet
    from voxmesh.data_io import synthesize_record
    from voxmesh.mesh import create_mesh
    from voxmesh.sharding import Layout

    E = 128
    cfg = unet.recipe_for_resolution(E, 0.125)
    g = {}
    with create_mesh([("one", 1)]) as mesh:
        graph = unet.build(cfg, mesh, Layout({}))
        params = unet.init_params(graph, 1)
    rec = synthesize_record(E, np.random.default_rng(np.random.SeedSequence([7, 0])), "case000")
    x = rec.image.astype(np.float64)[None, ..., None]
    oh = training.one_hot(rec.labels[None], 3).astype(np.float64)
    p64 = {k: {kk: vv.astype(np.float64) for kk, vv in v.items()} for k, v in params.items()}
    g["param_sum"] = np.array([sum(float(np.abs(v["kernel"]).sum()) for v in params.values())])
    t0 = time.time()
    probs, tape = oracle.oracle_forward(graph, p64, x)
    print(f"forward {time.time() - t0:.0f} s", flush=True)
    stats = training.loss_stats_local(probs, oh)
    rc = training._RunCtx(3, (1, 2), 0.9, 0.1, 1e-12, E ** 3, 0.0, 0.0, param_order=())
    g["loss_stats"] = np.asarray(stats, dtype=np.float64)
    g["loss_values"] = np.array(training.losses_from_stats(stats, rc), dtype=np.float64)
    idx = np.sort(np.random.default_rng(2024).choice(E ** 3, 32768, replace=False))
    g["probs_idx"] = idx.astype(np.int64)
    g["probs"] = probs.reshape(-1, 3)[idx]
    d = training.loss_grad_local(probs, oh, stats, rc)
    t0 = time.time()
    pg, _ = oracle.oracle_backward(graph, p64, tape, d)
    print(f"backward {time.time() - t0:.0f} s", flush=True)
    for nid, (gk, gb) in pg.items():
        g[f"gnorm_{nid}"] = np.array([np.linalg.norm(gk), np.linalg.norm(gb)])
        if nid in FULL_GRAD_LAYERS:
            g[f"gk_{nid}"] = gk.astype(np.float32)
            g[f"gb_{nid}"] = gb.astype(np.float32)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1024:.0f} KiB; loss {g['loss_values']}")


if __name__ == "__main__":
    main()
