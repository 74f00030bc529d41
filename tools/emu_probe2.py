"""Probe: does the emulated step slow down as training on one fixed sample diverges?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_03108_b200 as vm  # noqa: E402
from paper_1909_03108_b200.data import synth_record  # noqa: E402
from paper_1909_03108_b200.step import UNetStep  # noqa: E402

E, K = 256, 8
cfg = vm.recipe_for_resolution(E, 0.5)
mesh = vm.create_mesh([("one", 1)], backend="threads")
graph = vm.build(cfg, mesh, {})
loc = (E // K, E, E)
st = UNetStep(graph, vm.init_params(graph, 1), dtype=torch.bfloat16, global_shape=(E, E, E), local_shape=loc)
st.use_peer_halo(nbr6=[0, 0, -1, -1, -1, -1])
img, lab = synth_record(E, 7, 0)
st.upload(torch.from_numpy(img[None, :loc[0], ..., None].copy()), torch.from_numpy(lab[None, :loc[0]].copy()))
gs = {}
for on in (True, False):
    st.has_halo = on
    gs[on] = st.capture()
seq = [True] * 15 + [False] * 15 + [True] * 15
for i, on in enumerate(seq):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gs[on].replay()
    e1.record()
    e1.synchronize()
    fin = bool(torch.isfinite(st.params).all())
    print(f"{i:2d} halo={int(on)} {e0.elapsed_time(e1):7.3f} ms loss={st.loss()[0]:.4f} params_finite={fin} "
          f"skipped={int(st.skip_flags.sum())} maxabs={float(st.params.abs().max()):.3g}", flush=True)
