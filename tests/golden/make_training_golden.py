"""Generate the training-loop fixtures from the REFERENCE implementation (build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_training_golden.py

* ``ref_checkpoint/``: a checkpoint written by ``voxmesh.training.save_checkpoint``
  (training.py:414-428) for a small U-Net (params from ``init_params(graph, 1)``, moments
  0.5, extra {"note": "x"}), so tests check that our loader reads it and our writer
  produces the same files;
* ``training_golden.npz``: the record order ``BatchSource.batch`` visits (training.py:241-279)
  for seeds 0 and 11, 5 records, batch sizes 1 and 2, steps 0..11.
"""

import os
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from voxmesh import training, unet
    from voxmesh.data_io import VolumeRecord
    from voxmesh.mesh import create_mesh

    with create_mesh([("one", 1)]) as mesh:
        graph = unet.build(unet.UNetConfig(8, (4, 8), convs_per_block=1), mesh, {})
    params = unet.init_params(graph, 1)
    moments = {n: {k: np.full_like(v, 0.5) for k, v in b.items()} for n, b in params.items()}
    ck = os.path.join(HERE, "ref_checkpoint")
    shutil.rmtree(ck, ignore_errors=True)
    training.save_checkpoint(ck, 7, params, moments, extra={"note": "x"})

    out = {}
    recs = [VolumeRecord(np.full((2, 2, 2), float(i), np.float32), np.zeros((2, 2, 2), np.uint8), f"r{i}")
            for i in range(5)]
    for seed in (0, 11):
        for bs in (1, 2):
            src = training.BatchSource(recs, bs, seed, 3, np.float32)
            order = [[int(img[j, 0, 0, 0, 0]) for j in range(bs)] for img, _ in (src.batch(s) for s in range(12))]
            out[f"order_seed{seed}_bs{bs}"] = np.array(order, dtype=np.int64)
    np.savez(os.path.join(HERE, "training_golden.npz"), **out)
    print("wrote", ck, "and training_golden.npz:", sorted(out))


if __name__ == "__main__":
    main()
