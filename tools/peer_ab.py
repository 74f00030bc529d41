"""A/B of the emulated depth split (cfg3 K-way rank block, every neighbour = self): step time
with the peer-memory halo on / off, graph and eager, repeated in alternating order."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_03108_b200 as vm  # noqa: E402
from paper_1909_03108_b200.data import synth_record  # noqa: E402
from paper_1909_03108_b200.step import UNetStep  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
E = 256
cfg = vm.recipe_for_resolution(E, 0.5)
mesh = vm.create_mesh([("one", 1)], backend="threads")
graph = vm.build(cfg, mesh, {})
params = vm.init_params(graph, 1)
loc = (E // K, E, E)
st = UNetStep(graph, params, dtype=torch.bfloat16, global_shape=(E, E, E), local_shape=loc)
st.use_peer_halo(nbr6=[0, 0, -1, -1, -1, -1])
img, lab = synth_record(E, 7, 0)
st.upload(torch.from_numpy(img[None, :loc[0], ..., None].copy()), torch.from_numpy(lab[None, :loc[0]].copy()))
for _ in range(2):
    st.step()
torch.cuda.synchronize()


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


def variant(halo, graph_mode, wgrad_side=True):
    st.has_halo = halo
    st.overlap_wgrad = wgrad_side
    if not graph_mode:
        return timeit(st.step)
    g = st.capture()
    t = timeit(g.replay)
    del g
    return t


for rep in range(2):
    for halo in (True, False):
        print(f"rep {rep} halo={halo}: graph {variant(halo, True):.3f} ms  eager {variant(halo, False):.3f} ms  "
              f"graph no-side {variant(halo, True, False):.3f} ms", flush=True)
st.has_halo = True
st.halo.check()

# both programs captured first, then timed alternately (the bench.py pattern)
gs = {}
for halo in (True, False):
    st.has_halo = halo
    gs[halo] = st.capture()
for rep in range(2):
    for halo in (True, False):
        print(f"both-captured rep {rep} halo={halo}: {timeit(gs[halo].replay):.3f} ms", flush=True)
del gs
gs = {}
for halo in (False, True):
    st.has_halo = halo
    gs[halo] = st.capture()
for halo in (True, False):
    print(f"both-captured (nohalo first) halo={halo}: {timeit(gs[halo].replay):.3f} ms", flush=True)
