"""Critical-path probe of the cfg2 train step (diagnostic, not a bench number): graph-replay
time of the full step and of variants that drop or serialise parts of it.

    full            forward + backward (wgrad on the side stream) + SGD + repack
    serial_wgrad    same, wgrad on the main stream
    no_wgrad        main stream only (weight gradients skipped)   -- INVALID as a step
    fwd_only        forward (+ loss statistics)
    wgrad_only      the weight-gradient launches alone, back to back
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1909_03108_b200 as vm  # noqa: E402
from paper_1909_03108_b200 import _lib  # noqa: E402
from paper_1909_03108_b200.data import synth_record  # noqa: E402
from paper_1909_03108_b200.step import UNetStep  # noqa: E402

pdl = int(os.environ.get("PDL_FWD", "1"))
cfg = vm.recipe_for_resolution(128, 1 / 8)
mesh = vm.create_mesh([("one", 1)], backend="threads")
graph = vm.build(cfg, mesh, {})
st = UNetStep(graph, vm.init_params(graph, 1), batch=1, ctx=None, dtype=torch.bfloat16)
im, lb = synth_record(128, 7, 0)
st.upload(torch.from_numpy(im[None, ..., None].copy()), torch.from_numpy(lb[None].copy()))
st.pdl_forward = pdl
st.pdl_backward = int(os.environ.get("PDL_BWD", "2"))
st.step()
torch.cuda.synchronize()


def _capture(fn):
    import gc

    gc.collect()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    return g


def timed(fn, reps=30):
    g = _capture(fn)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
res["full"] = timed(st.step)
st.overlap_wgrad = False
res["serial_wgrad"] = timed(st.step)
st.overlap_wgrad = True
real = st._wgrad
st._wgrad = lambda *a, **k: None
res["no_wgrad"] = timed(st.step)
st._wgrad = real


def fwd():
    st.forward()


res["fwd_only"] = timed(fwd)
calls = []
st._wgrad = lambda *a, **k: calls.append(a)
st.backward()
torch.cuda.synchronize()
st._wgrad = real


def wg():
    for a in calls:
        real(*a)


res["wgrad_only"] = timed(wg)
_lib.load().vm_debug_skip_wgrad_finalize(1)
res["wgrad_only_nofin"] = timed(wg)
res["full_nofin"] = timed(st.step)
_lib.load().vm_debug_skip_wgrad_finalize(0)
print(f"pdl_forward={pdl} pdl_backward={int(st.pdl_backward)} " + " ".join(f"{k}={v:.3f}ms" for k, v in res.items()))
