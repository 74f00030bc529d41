"""Run ONE eager cfg2 train step inside a cudaProfilerStart/Stop window, for
``ncu --profile-from-start off -k regex:^k_ --set full``.  Writes the per-call launch
map (kind, layer, number of kernels the call launched) to ``--map`` so that
``tools/ncu_summary.py --map`` can attribute every profiled launch to its step op.

    ncu --profile-from-start off -k regex:^k_ --set full --clock-control none \
        --import-source on -o gpurun_out/step_full python tools/ncu_step.py --map gpurun_out/step_map.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--extent", type=int, default=128)
    ap.add_argument("--scale", type=float, default=1 / 8)
    ap.add_argument("--map", default="gpurun_out/step_map.json")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_1909_03108_b200 as vm
    from paper_1909_03108_b200 import _lib
    from paper_1909_03108_b200.data import synth_record
    from paper_1909_03108_b200.step import UNetStep

    cfg = vm.recipe_for_resolution(a.extent, a.scale)
    mesh = vm.create_mesh([("one", 1)], backend="threads")
    graph = vm.build(cfg, mesh, {})
    st = UNetStep(graph, vm.init_params(graph, 1), batch=1, ctx=None, dtype=torch.bfloat16)
    im, lb = synth_record(a.extent, 7, 0)
    st.upload(torch.from_numpy(im[None, ..., None].copy()), torch.from_numpy(lb[None].copy()))
    for _ in range(2):
        st.step()
    # record the launch list of one step, then replay it call by call under the profiler
    st._rec = []
    st.step()
    rec, st._rec = st._rec, None
    torch.cuda.synchronize()
    lib = _lib.load()
    calls = []
    torch.cuda.cudart().cudaProfilerStart()
    for kind, label, flops, nbytes, name, args in rec:
        n0 = lib.vm_launch_count()
        _lib.call(name, *args, _lib.stream_ptr())
        calls.append({"kind": kind, "layer": label, "flops": flops, "bytes": nbytes, "fn": name,
                      "kernels": lib.vm_launch_count() - n0})
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    os.makedirs(os.path.dirname(os.path.abspath(a.map)), exist_ok=True)
    json.dump(calls, open(a.map, "w"), indent=1)
    print(f"{len(calls)} calls, {sum(c['kernels'] for c in calls)} kernels")


if __name__ == "__main__":
    main()
