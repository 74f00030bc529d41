#!/usr/bin/env python
"""Benchmark: spatially partitioned 3D U-Net train step on B200 (voxels/s).

Workload (BASELINE.json configs[1], "cfg2"): U-Net recipe_for_resolution(128, 1/8)
= filters (16, 32, 64, 128), 4 conv per block, 128^3 synthetic CT volume, batch 1,
bf16 storage / fp32 accumulation, SGD momentum step included.  With N GPUs
(torchrun, one process per GPU) the volume grows along depth to (128 N) x 128 x 128
and is depth-split over a 1-D mesh — fixed per-GPU work (weak scaling) with a halo
exchange before every 3x3x3 conv, forward and backward, and the weight-gradient
all-reduce.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the CPU oracle port of
the reference (oracle/voxmesh_oracle.py) on a bounded sample instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3D U-Net train voxels/sec at 1/2/4/8 B200; halo-exchange % of step time"
PEAKS = {"hbm_gbs": 6552.0, "bf16_tflops": 1658.2, "bf16_tflops_sustained": 1381.0}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {k: float(d[k]) for k in PEAKS}, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback (B200_PROFILING.md)"


def load_traffic(kind):
    """roofline.traffic: DRAM bytes (read+write) per launch of ``kind``, from the newest
    committed ncu step capture (dram__bytes_read.sum + dram__bytes_write.sum per launch) (profiles/r*/ncu_step_dram.json, written by
    tools/ncu_summary.py --map); None when no capture is committed."""
    import glob

    caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_step_dram.json")))
    if not caps:
        return None, None
    try:
        by = json.load(open(caps[-1]))["by_kind"]
        return by[kind]["dram_bytes_per_call"], os.path.relpath(caps[-1], ROOT)
    except Exception:
        return None, os.path.relpath(caps[-1], ROOT)


def _capture(torch, fn):
    """Capture ``fn`` as one CUDA graph on a side stream; None if capture fails (e.g. a
    collective that cannot be captured), in which case the step runs eagerly."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                fn()
    except Exception as e:  # pragma: no cover - GPU path
        print(f"[bench] CUDA graph capture failed ({e}); running eagerly", file=sys.stderr)
        torch.cuda.synchronize()
        return None
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return g


def args_parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--conv", default="tc", choices=["tc", "simt"])
    p.add_argument("--extent", type=int, default=128)
    p.add_argument("--scale", type=float, default=0.125)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--graph-multi", action="store_true",
                   help="also capture the step as a CUDA graph when N > 1 (NCCL halo inside the graph)")
    p.add_argument("--cpu-sample-extent", type=int, default=32)
    p.add_argument("--layer-csv", default=None, help="write per-layer kernel times here")
    return p.parse_args()


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML while the timed region runs."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {
            "sm_mhz": statistics.median(self.samples),
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


# ---------------------------------------------------------------------- CPU legs
def cpu_sample(extent, scale, steps=1):
    """Time the oracle port (numpy) of the same network on a bounded extent^3 sample."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import voxmesh_oracle as O

    filters = O.recipe_filters(128, scale)  # the cfg2 network
    nodes = O.graph_nodes(filters)
    params = O.init_params(nodes, 1)
    moments = {k: {kk: np.zeros_like(vv) for kk, vv in v.items()} for k, v in params.items()}
    img, lab = O.record_for(extent, 0)
    x = img[None, ..., None]
    oh = O.one_hot(lab[None], 3)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.train_step(nodes, params, moments, x, oh)
        times.append(time.perf_counter() - t0)
    per = min(times)
    try:
        from threadpoolctl import threadpool_info

        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count() or 1
    return extent ** 3 / per, per, cores


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    cores = 1
    for _ in range(max(1, a.warmup // 3)):
        cpu_sample(a.cpu_sample_extent, a.scale)
    for _ in range(a.steps):
        v, per, cores = cpu_sample(a.cpu_sample_extent, a.scale)
        vals.append(v)
    value = statistics.median(vals)
    sample = (f"oracle port (numpy, oracle/voxmesh_oracle.py) fwd+bwd+SGD of the cfg2 network "
              f"{a.cpu_sample_extent}^3 x 1 per step (bounded sample of the 128^3 workload)")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "voxels/s",
        "n_gpus": a.gpus,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": 1e3 * a.cpu_sample_extent ** 3 / value,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (data_io.synthesize_record distribution, SeedSequence([7, 0]))",
        "config": {"workload": "cfg2 network recipe_for_resolution(128, 1/8), CPU bounded sample",
                   "global_batch": 1, "sample_extent": a.cpu_sample_extent},
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- GPU leg
def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1909_03108_b200 as vm
    from paper_1909_03108_b200 import _lib
    from paper_1909_03108_b200.data import synth_record
    from paper_1909_03108_b200.step import UNetStep

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peak_src = load_peaks()

    cfg = vm.recipe_for_resolution(a.extent, a.scale)
    E = a.extent
    if world > 1:
        mesh = vm.create_mesh([("mx", world)])
        layout = {"x": "mx"}
    else:
        mesh = vm.create_mesh([("one", 1)], backend="threads")
        layout = {}
    graph = vm.build(cfg, mesh, layout)
    params = vm.init_params(graph, 1)
    ctx = mesh.context(rank) if world > 1 else None
    # weak scaling: each rank owns one E^3 block of a (E*world) x E x E volume
    st = UNetStep(graph, params, batch=a.batch, ctx=ctx, dtype=torch.bfloat16, conv_impl=a.conv,
                  global_shape=(E * world, E, E), local_shape=(E, E, E))
    imgs, labs = [], []
    for b in range(a.batch):
        im, lb = synth_record(E, 7, rank * a.batch + b)
        imgs.append(im)
        labs.append(lb)
    img_h = torch.from_numpy(np.stack(imgs)[..., None].copy()).pin_memory()
    lab_h = torch.from_numpy(np.stack(labs).copy()).pin_memory()
    st.upload(img_h, lab_h)
    torch.cuda.synchronize()

    # warm-up (eager), then capture the step as one CUDA graph
    for _ in range(max(1, min(2, a.warmup))):
        st.step()
    torch.cuda.synchronize()
    l0 = _lib.load().vm_launch_count()
    st.step()
    torch.cuda.synchronize()
    launches_per_step = _lib.load().vm_launch_count() - l0
    graph_obj = None
    graph_note = "disabled (--no-graph)" if a.no_graph else "captured"
    if world > 1 and not a.graph_multi and not a.no_graph:
        # the NCCL halo groups are not validated inside CUDA graphs on multi-GPU hardware yet:
        # eager launches (measured 8% slower at N = 1)
        a.no_graph = True
        graph_note = "eager (N > 1: NCCL halo not captured; --graph-multi to capture)"
    if not a.no_graph:
        graph_obj = _capture(torch, st.step)
        if graph_obj is None:
            graph_note = "capture failed, eager launches"

    def one():
        if graph_obj is not None:
            graph_obj.replay()
        else:
            st.step()

    for _ in range(a.warmup):
        one()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: device-resident inputs
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(a.steps):
            one()
        e1.record()
        e1.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    voxels = a.batch * world * E ** 3
    value = voxels / (ms * 1e-3)

    # ---- end-to-end through the public API: host buffers, H2D + D2H inside the timed region
    # every step: H2D of its inputs (step k+1's overlapping step k on a copy stream) and an
    # async D2H of its loss statistics, read by the host while the next step runs.  The path
    # is warmed up first (pinned staging buffers, copy stream, events), like the device loop.
    st.train_loop_host([(img_h, lab_h)] * max(a.warmup, 1), replay=one)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    losses = st.train_loop_host([(img_h, lab_h)] * a.steps, replay=one)
    loss = losses[-1][0]
    f1.record()
    f1.synchronize()
    barrier()
    ms_e2e = f0.elapsed_time(f1) / a.steps
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    h2d = img_h.numel() * img_h.element_size() + lab_h.numel() * lab_h.element_size()
    d2h = st.stats.numel() * 4

    # ---- halo share (A/B, the paper's "adds around 5%")
    halo = {"share": 0.0, "method": "A/B: (t_step - t_step_nohalo)/t_step", "bytes_per_step_rank": 0}
    if world > 1:
        st.has_halo_saved = st.has_halo
        st.has_halo = False
        g2 = _capture(torch, st.step) if graph_obj is not None else None
        run2 = g2.replay if g2 is not None else st.step
        for _ in range(a.warmup):
            run2()
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record()
        for _ in range(a.steps):
            run2()
        h1.record()
        h1.synchronize()
        ms_nohalo = h0.elapsed_time(h1) / a.steps
        t = torch.tensor([ms_nohalo], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_nohalo = float(t.item())
        st.has_halo = st.has_halo_saved
        halo["share"] = max(0.0, (ms - ms_nohalo) / ms)
        halo["ms_nohalo"] = ms_nohalo
        halo["bytes_per_step_rank"] = st.halo_bytes_per_step()

    # ---- per-kernel timing for the roofline (each launch replayed alone as a CUDA graph)
    prof = st.profile_kernels(reps=5)
    classes = {}
    for row in prof:
        c = classes.setdefault(row["kind"], {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0})
        c["ms"] += row["ms"]
        c["flops"] += row["flops"]
        c["bytes"] += row["bytes"]
        c["launches"] += 1
    dom_kind = max(classes, key=lambda k: classes[k]["ms"])
    dom = classes[dom_kind]
    step_kernel_ms = sum(c["ms"] for c in classes.values())
    traffic, traffic_src = load_traffic(dom_kind)
    if dom["flops"] > 0:
        achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["bf16_tflops"], "traffic": traffic}
    else:
        achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic}
    roof.update({"kernel": dom_kind, "launches_per_step": dom["launches"],
                 "algorithmic_bytes_per_launch": dom["bytes"] / max(dom["launches"], 1),
                 "flops_per_launch": dom["flops"] / max(dom["launches"], 1),
                 "avg_launch_ms": dom["ms"] / max(dom["launches"], 1),
                 "share_of_kernel_time": dom["ms"] / step_kernel_ms, "peak_source": peak_src,
                 "traffic_source": traffic_src})
    conv_flops = graph.conv_flops(a.batch) * (world * E ** 3) / (E ** 3) / world  # per rank
    cfg_name = {(128, 0.125): "cfg2", (256, 0.5): "cfg3", (512, 1.0): "cfg4"}.get((E, a.scale), "custom")
    act_gb = torch.cuda.memory_allocated() / 1e9  # activation slabs, tape, grads, workspaces
    conv_ms = sum(c["ms"] for k, c in classes.items() if k.startswith("conv"))
    if a.layer_csv and rank == 0:
        with open(a.layer_csv, "w") as f:
            f.write("layer,kind,ms,flops,bytes,tflops,gbs\n")
            for r in prof:
                f.write(f"{r['layer']},{r['kind']},{r['ms']:.4f},{r['flops']:.0f},{r['bytes']:.0f},"
                        f"{r['flops'] / max(r['ms'], 1e-9) / 1e9:.1f},{r['bytes'] / max(r['ms'], 1e-9) / 1e6:.1f}\n")

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    try:
        v, per, cores = cpu_sample(a.cpu_sample_extent, a.scale)
        cpu = {"value": v, "unit": "voxels/s", "cores": cores, "kind": "port",
               "sample": f"oracle port fwd+bwd+SGD of the cfg2 network on a {a.cpu_sample_extent}^3 volume, 1 step "
                         f"({per:.1f} s)"}
    except Exception as e:  # pragma: no cover
        cpu = {"value": None, "unit": "voxels/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "voxels/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (data_io.synthesize_record distribution, SeedSequence([7, rank]))",
        "config": {
            "workload": f"{cfg_name}: U-Net recipe_for_resolution({E}, {a.scale:g}) = {cfg.encoder_filters}, "
                        f"{E}^3 per GPU, batch {a.batch}" + (f", depth-split x{world}" if world > 1 else ""),
            "global_batch": a.batch,
            "volume": [E * world, E, E],
            "parallelism": f"spatial depth-split x{world}" if world > 1 else "single GPU",
            "conv": a.conv,
            "cuda_graph": graph_note,
            "l2": f"working set (activation slabs, {act_gb:.1f} GB) >> 126 MB L2; no flush needed",
            "conv_tflop_per_step_rank": conv_flops / 1e12,
        },
        "e2e": {"value": voxels / (ms_e2e * 1e-3), "unit": "voxels/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e, "loss": loss,
                "path": "UNetStep.train_loop_host: per step pinned H2D (prefetched one step ahead on a copy "
                        "stream) -> slab/one-hot kernels -> step graph -> async D2H of the loss statistics"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * a.steps,
        "halo": halo,
        "kernel_ms_per_step": {k: round(c["ms"], 4) for k, c in classes.items()},
        # every kernel class against its own roofline (tensor for convs, HBM for the rest),
        # each launch replayed alone: the dominant class above is one row of this table
        "roofline_by_kind": {
            k: ({"bound": "tensor", "tflops": round(c["flops"] / (c["ms"] * 1e-3) / 1e12, 1),
                 "frac": round(c["flops"] / (c["ms"] * 1e-3) / 1e12 / peaks["bf16_tflops"], 3)}
                if c["flops"] > 0 and k.startswith("conv") else
                {"bound": "hbm", "gbs": round(c["bytes"] / (c["ms"] * 1e-3) / 1e9, 0),
                 "frac": round(c["bytes"] / (c["ms"] * 1e-3) / 1e9 / peaks["hbm_gbs"], 3)})
            for k, c in classes.items() if c["ms"] > 0},
        "conv_tflops_effective": conv_flops / (conv_ms * 1e-3) / 1e12 if conv_ms else None,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = args_parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
