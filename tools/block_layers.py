"""Per-layer kernel times of one rank's block of a depth split (default cfg3 8-way: 32x256x256),
each launch replayed alone; grouped by level and kind.  Args: [ways [extent [scale]]]
(cfg2: ``1 128 0.125``)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_03108_b200 as vm  # noqa: E402
from paper_1909_03108_b200.data import synth_record  # noqa: E402
from paper_1909_03108_b200.step import UNetStep  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
E = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = vm.recipe_for_resolution(E, float(sys.argv[3]) if len(sys.argv) > 3 else 0.5)
mesh = vm.create_mesh([("one", 1)], backend="threads")
graph = vm.build(cfg, mesh, {})
loc = (E // K, E, E)
st = UNetStep(graph, vm.init_params(graph, 1), dtype=torch.bfloat16, global_shape=(E, E, E), local_shape=loc)
img, lab = synth_record(E, 7, 0)
st.upload(torch.from_numpy(img[None, :loc[0], ..., None].copy()), torch.from_numpy(lab[None, :loc[0]].copy()))
st.step()
torch.cuda.synchronize()
rows = st.profile_kernels(reps=5)
by = {}
for r in rows:
    lay = r["layer"]
    lvl = lay[:4] if lay[:3] in ("enc", "dec") else lay
    k = (lvl, r["kind"])
    b = by.setdefault(k, [0.0, 0.0, 0])
    b[0] += r["ms"]
    b[1] += r["flops"]
    b[2] += 1
tot = sum(v[0] for v in by.values())
print(f"block {loc}: sum of launches {tot:.3f} ms")
for k, v in sorted(by.items(), key=lambda kv: -kv[1][0])[:28]:
    print(f"{k[0]:6s} {k[1]:11s} n={v[2]:2d} {v[0] * 1e3:8.1f} us {v[1] / max(v[0], 1e-9) / 1e9:7.1f} TF/s")
for r in sorted(rows, key=lambda r: -r["ms"])[:16]:
    print(f"  {r['layer']:12s} {r['kind']:11s} {r['ms'] * 1e3:7.1f} us {r['flops'] / max(r['ms'], 1e-9) / 1e9:7.1f} TF/s")
for k, v in sorted(by.items()):
    if k[1] in ("head_fwd", "head_bwd", "pool_fwd", "pool_bwd", "up_fwd", "up_bwd", "sgd", "pack"):
        print(f"  {k[0]:6s} {k[1]:11s} {v[0] * 1e3:8.1f} us")
