"""Probe: bench.emulated_halo alone (no cfg2 run before it) vs after a cfg2 step object exists."""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_03108_b200 as vm  # noqa: E402

a = types.SimpleNamespace(emulate_split=8, emulate_transport="peer", no_graph=False, warmup=3, steps=10)
peaks, _ = bench.load_peaks()
r = bench.emulated_halo(a, torch, vm, peaks)
print("alone:", r["ms_step"], r["ms_nohalo"], r["share"], r["rounds_ms"], flush=True)
a.warmup = 20
r = bench.emulated_halo(a, torch, vm, peaks)
print("warmup 20:", r["ms_step"], r["ms_nohalo"], r["share"], r["rounds_ms"], flush=True)
if len(sys.argv) > 1:
    from paper_1909_03108_b200.step import UNetStep
    cfg = vm.recipe_for_resolution(128, 0.125)
    mesh = vm.create_mesh([("one", 1)], backend="threads")
    graph = vm.build(cfg, mesh, {})
    st = UNetStep(graph, vm.init_params(graph, 1), dtype=torch.bfloat16)
    g = st.capture()
    g.replay()
    torch.cuda.synchronize()
    r = bench.emulated_halo(a, torch, vm, peaks)
    print("after cfg2 graph:", r["ms_step"], r["ms_nohalo"], r["share"], flush=True)
