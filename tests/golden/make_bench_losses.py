"""Oracle losses of the bench workloads' FIRST step (fresh init_params(seed 1), record i of
dataset seed 7 for sample i), so bench.py can assert its own first-step loss.

    python tests/golden/make_bench_losses.py            # writes tests/golden/bench_losses.json

cfg2 comes from the reference's own f64 network (tests/golden/cfg2_golden.npz).  cfg3
(recipe_for_resolution(256, 0.5) at 256^3) is too large for the reference's einsum network
or an f64 tape in this container's RAM, so it runs the oracle port (oracle/voxmesh_oracle.py,
pinned to the reference by tests/golden/) in float32 with a streaming forward that keeps
only the skip tensors; the f32 oracle's loss error (~1e-6) is far below the 1e-2 gate.
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import voxmesh_oracle as O  # noqa: E402

OUT = os.path.join(HERE, "bench_losses.json")


def streaming_loss(extent, scale, batch=1, dtype=np.float32):
    filters = O.recipe_filters(extent, scale)
    nodes = O.graph_nodes(filters)
    params = O.init_params(nodes, 1)
    consumers = {}
    for nid, op, inputs, *_ in nodes:
        for i in inputs:
            consumers[i] = consumers.get(i, 0) + 1
    stats = None
    for b in range(batch):
        img, lab = O.record_for(extent, b)
        acts = {"input": img[None, ..., None].astype(dtype)}
        left = dict(consumers)
        for nid, op, inputs, k, ci, co in nodes:
            a = acts[inputs[0]]
            if op == "conv":
                out = O.conv3d_dense(a, params[nid]["kernel"].astype(dtype), params[nid]["bias"].astype(dtype))
            elif op == "relu":
                out = np.maximum(a, 0, out=a if left[inputs[0]] == 1 else None)
            elif op == "pool":
                out, _ = O.maxpool2_dense(a)
            elif op == "up":
                out = O.upsample2_dense(a)
            elif op == "concat":
                out = np.concatenate([a, acts[inputs[1]]], axis=-1)
            elif op == "softmax":
                out = O.softmax_dense(a)
            acts[nid] = out
            for i in inputs:
                left[i] -= 1
                if left[i] == 0 and i in acts:
                    del acts[i]
        probs = acts[nodes[-1][0]]
        s = O.loss_stats(probs.astype(np.float64), O.one_hot(lab[None], 3).astype(np.float64))
        stats = s if stats is None else stats + s
    return O.losses_from_stats(stats, 3, batch * extent ** 3), len(params)


def main():
    out = {}
    gold = np.load(os.path.join(HERE, "cfg2_golden.npz"))
    out["cfg2"] = {"loss": float(gold["loss_values"][0]), "source": "reference f64 network (cfg2_golden.npz)"}
    t0 = time.time()
    (loss, dice, ce), _ = streaming_loss(256, 0.5)
    out["cfg3"] = {"loss": float(loss), "dice": float(dice), "ce": float(ce),
                   "source": f"oracle port f32 streaming forward ({time.time() - t0:.0f} s)"}
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
