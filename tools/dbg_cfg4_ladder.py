"""Per-layer gradient differences: cfg4 ladder at 64^3, 2x2x2 threads mesh vs one rank vs the f64 oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200.step import UNetStep
from tests.helpers import node_tuples, rel_l2
from tests.test_gpu_configs import _cfg4_small, _run_partitioned

E = int(sys.argv[1]) if len(sys.argv) > 1 else 64
axes = [("mx", 2), ("my", 2), ("mz", 2)]
layout = {"x": "mx", "y": "my", "z": "mz"}
cfg = _cfg4_small(E)
m1 = vm.create_mesh([("one", 1)])
g1 = vm.build(cfg, m1, {})
params = vm.init_params(g1, 2)
img, lab = O.record_for(E, 0)
img, lab = img[None, ..., None].astype(np.float32), lab[None].astype(np.uint8)
st = UNetStep(g1, params, batch=1, dtype=torch.bfloat16, device="cuda")
st.upload(torch.from_numpy(img), torch.from_numpy(lab))
st.forward(); st.backward(); torch.cuda.synchronize()
grads1 = st.grad_dict()
g, res = _run_partitioned(cfg, params, axes, layout, img, lab)
p64 = {k: {kk: np.asarray(vv, np.float64) for kk, vv in v.items()} for k, v in params.items()}
nodes = node_tuples(g1)
probs, tape, _ = O.oracle_forward(nodes, p64, img.astype(np.float64))
oh = O.one_hot(lab, 3).astype(np.float64)
stats = O.loss_stats(probs, oh)
d = O.loss_grad(probs, oh, stats, E ** 3)
rg, _ = O.oracle_backward(nodes, p64, tape, d)
print(f"{'layer':14s} {'part-vs-1':>10s} {'1-vs-f64':>10s} {'part-vs-f64':>11s}  ext")
for L in st.layers:
    k = L.node.id
    a = rel_l2(res[0][1][k][0], grads1[k][0]); b = rel_l2(grads1[k][0], rg[k][0]); c = rel_l2(res[0][1][k][0], rg[k][0])
    print(f"{k:14s} {a:10.2e} {b:10.2e} {c:11.2e}  {L.D}x{L.H}x{L.W} {L.cin}->{L.cout}")
