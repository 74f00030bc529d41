"""Per-step timeline of the public-API train loop (train_loop_host) vs device-only replays."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
import paper_1909_03108_b200 as vm  # noqa: E402
from paper_1909_03108_b200.data import synth_record  # noqa: E402
from paper_1909_03108_b200.step import UNetStep  # noqa: E402

E = 128
cfg = vm.recipe_for_resolution(E, 1 / 8)
mesh = vm.create_mesh([("one", 1)], backend="threads")
graph = vm.build(cfg, mesh, {})
st = UNetStep(graph, vm.init_params(graph, 1), dtype=torch.bfloat16)
im, lb = synth_record(E, 7, 0)
img_h = torch.from_numpy(im[None, ..., None].copy()).pin_memory()
lab_h = torch.from_numpy(lb[None].copy()).pin_memory()
st.upload(img_h, lab_h)
for _ in range(3):
    st.step()
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        st.step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
for rep in range(4):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = st.train_loop_host([(img_h, lab_h)] * 50, replay=g.replay)
    e1.record()
    e1.synchronize()
    t1 = time.perf_counter()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(50):
        g.replay()
    e3.record()
    e3.synchronize()
    print(f"rep {rep}: e2e {e0.elapsed_time(e1) / 50:.3f} ms/step (host {1e3 * (t1 - t0) / 50:.3f}), "
          f"graph only {e2.elapsed_time(e3) / 50:.3f} ms/step")
