#!/usr/bin/env python
"""Benchmark: spatially partitioned 3D U-Net train step on B200 (voxels/s; halo share).

Workloads (BASELINE.json configs):
  cfg2  recipe_for_resolution(128, 1/8) = (16, 32, 64, 128), 128^3, batch 1, one GPU
        (the default at N = 1: BASELINE.json configs[1]);
  cfg3  recipe_for_resolution(256, 0.5) = (32 .. 512), 256^3, batch 1, depth split over the
        N GPUs (strong scaling; the default at N > 1);
  cfg4  recipe_for_resolution(512, 1.0) = (32 .. 1024), 512^3, batch 1, 2x2x2 mesh (N = 8);
  cfg5  the cfg4 network, 512^3, global batch 2, mesh b=2 x mx=2 x my=2 (N = 8).
bf16 storage / fp32 accumulation, SGD with momentum inside every step; synthetic CT volumes
(data_io.synthesize_record distribution) and init_params(seed 1).  One process per GPU
(torchrun); the halo is NCCL send/recv through the C ABI (vm_halo_slab_fwd) and the weight
gradients are all-reduced in buckets on a second communicator, the whole step captured in one
CUDA graph (``--no-graph`` for eager launches).

Before timing, the first step's loss is checked against the stored oracle loss of the same
inputs (tests/golden/bench_losses.json) and the run aborts on a mismatch.

At N = 1 the halo share is measured by emulation: one rank's block of cfg3's 8-way depth
split runs with periodic halos (every neighbour = this rank) through the peer-memory depth
halo (vm_halo_depth_push: the same launches, fences and flags as a real split, local HBM
instead of NVLink wire time, which is reported separately as bytes / 770 GB/s), A/B against
the same block with the exchange switched off (``--emulate-transport nccl``: pack / 1-rank
NCCL group / unpack instead).

Prints ONE JSON line (rank 0).  ``--impl reference`` times the CPU oracle port of the
reference (oracle/voxmesh_oracle.py) on the same config instead.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3D U-Net train voxels/sec at 1/2/4/8 B200; halo-exchange % of step time"
PEAKS = {"hbm_gbs": 6552.0, "bf16_tflops": 1658.2, "bf16_tflops_sustained": 1381.0}
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal

CONFIGS = {
    "cfg2": dict(extent=128, scale=0.125, batch=1, mesh=lambda n: [("mx", n)] if n > 1 else [],
                 layout=lambda n: {"x": "mx"} if n > 1 else {}),
    "cfg3": dict(extent=256, scale=0.5, batch=1, mesh=lambda n: [("mx", n)] if n > 1 else [],
                 layout=lambda n: {"x": "mx"} if n > 1 else {}),
    "cfg4": dict(extent=512, scale=1.0, batch=1, mesh=lambda n: [("mx", 2), ("my", 2), ("mz", 2)],
                 layout=lambda n: {"x": "mx", "y": "my", "z": "mz"}, gpus=8),
    "cfg5": dict(extent=512, scale=1.0, batch=2, mesh=lambda n: [("b", 2), ("mx", 2), ("my", 2)],
                 layout=lambda n: {"batch": "b", "x": "mx", "y": "my"}, gpus=8),
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {k: float(d[k]) for k in PEAKS}, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback (B200_PROFILING.md)"


def load_traffic(kind, cfg_name):
    """roofline.traffic: DRAM bytes (read+write) per launch of ``kind`` from a committed ncu
    capture of the SAME config (profiles/r*/ncu_step_dram_<cfg>.json), else None."""
    import glob

    caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_step_dram_{cfg_name}.json")))
    if not caps:
        return None, None
    try:
        by = json.load(open(caps[-1]))["by_kind"]
        return by[kind]["dram_bytes_per_call"], os.path.relpath(caps[-1], ROOT)
    except Exception:
        return None, os.path.relpath(caps[-1], ROOT)


def args_parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="auto", choices=["auto"] + sorted(CONFIGS))
    p.add_argument("--conv", default="tc", choices=["tc", "simt"])
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of the captured step graph")
    p.add_argument("--no-emulate", action="store_true", help="N = 1: skip the emulated-split halo measurement")
    p.add_argument("--emulate-split", type=int, default=8, help="N = 1: depth split whose rank block is emulated")
    p.add_argument("--no-emulate-cfg4", action="store_true", help="N = 1: skip the cfg4 / cfg5 rank-block emulations")
    p.add_argument("--emulate-config", default="cfg3", choices=["cfg3", "cfg4", "cfg5"],
                   help="N = 1: cfg3 depth-split rank block, or one rank block of cfg4's 2x2x2 / cfg5's b x 2x2 mesh (NCCL)")
    p.add_argument("--emulate-transport", default="peer", choices=["peer", "nccl"],
                   help="N = 1: halo transport of the emulated split")
    p.add_argument("--halo-transport", default="peer", choices=["peer", "nccl"],
                   help="N > 1, depth-only split: peer-memory pushes (CUDA IPC) or NCCL send/recv")
    p.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    p.add_argument("--cpu-budget", type=float, default=150.0, help="seconds of CPU-oracle time (reference arm)")
    p.add_argument("--layer-csv", default=None, help="write per-layer kernel times here")
    p.add_argument("--scaling-base", default="auto", choices=["auto", "on", "off"],
                   help="cfg3: also time the unpartitioned network on rank 0's GPU alone (auto: at N > 1)")
    a = p.parse_args()
    if a.config == "auto":
        a.config = "cfg2" if a.gpus == 1 else "cfg3"
    need = CONFIGS[a.config].get("gpus")
    if need and a.gpus != need:
        p.error(f"{a.config} runs on exactly {need} GPUs (its mesh), got --gpus {a.gpus}")
    return a


def workload(a):
    c = CONFIGS[a.config]
    E, n = c["extent"], a.gpus
    mesh = c["mesh"](n)
    par = "x".join(f"{ax}{s}" for ax, s in mesh) if mesh else "single GPU"
    return {
        "workload": f"{a.config}: U-Net recipe_for_resolution({E}, {c['scale']:g}), {E}^3 volume, "
                    f"global batch {c['batch']}" + (f", spatial mesh {par}" if mesh else ", one GPU"),
        "global_batch": c["batch"],
        "volume": [E, E, E],
        "parallelism": par,
    }


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
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------- CPU legs
def _cpu_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_sample(config, budget_s, min_steps=1, max_steps=None):
    """Time the oracle port (numpy, the reference's algorithm) on ``config``'s network.  cfg2:
    full 128^3 steps (~30 s each on 16 host threads); the 256^3 / 512^3 configs: a
    16 x 128 x 128 sub-volume per step (the full step is hours).  Steps until ``budget_s``."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import voxmesh_oracle as O

    c = CONFIGS[config]
    filters = O.recipe_filters(c["extent"], c["scale"])
    nodes = O.graph_nodes(filters)
    params = O.init_params(nodes, 1)
    moments = {k: {kk: np.zeros_like(vv) for kk, vv in v.items()} for k, v in params.items()}
    if config == "cfg2":
        img, lab = O.record_for(128, 0)
        shape = (128, 128, 128)
    else:
        img, lab = O.record_for(128, 0)
        img, lab = img[56:72], lab[56:72]
        shape = (16, 128, 128)
    x = img[None, ..., None].astype(np.float32)
    oh = O.one_hot(lab[None], 3)
    times = []
    t_start = time.perf_counter()
    while len(times) < min_steps or (time.perf_counter() - t_start < budget_s and (max_steps is None or
                                                                                 len(times) < max_steps)):
        t0 = time.perf_counter()
        O.train_step(nodes, params, moments, x, oh)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start + times[-1] > budget_s and len(times) >= min_steps:
            break
    per = statistics.median(times)
    vox = shape[0] * shape[1] * shape[2]
    sample = (f"oracle port (oracle/voxmesh_oracle.py, numpy f32) fwd+bwd+SGD of the {config} network "
              f"recipe_filters={filters} on a {shape[0]}x{shape[1]}x{shape[2]} volume"
              + (" (the full workload)" if config == "cfg2" else " (bounded sub-volume of the workload)")
              + f", {len(times)} step(s), median {per:.1f} s")
    return vox / per, per, _cpu_threads(), sample, len(times)


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    value, per, cores, sample, n = cpu_sample(a.config, a.cpu_budget)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "voxels/s",
        "n_gpus": a.gpus,
        "steps": n,
        "warmup": 0,
        "ms_per_step": per * 1e3,
        "higher_is_better": True,
        "scaling": "strong" if a.gpus > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (data_io.synthesize_record distribution, SeedSequence([7, 0]))",
        "config": workload(a),
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": f"{n} timed step(s) of the requested {a.steps} (CPU time budget {a.cpu_budget:.0f} s)",
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- GPU leg
def _capture(torch, st, allow):
    if not allow:
        return None, "disabled (--no-graph)"
    try:
        g = st.capture()
    except Exception as e:  # pragma: no cover - GPU path
        print(f"[bench] !!! CUDA graph capture FAILED ({e}); running EAGER launches", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        return None, f"capture failed ({type(e).__name__}), eager launches"
    if g is None:
        print("[bench] !!! step not capturable with this transport; running EAGER launches", file=sys.stderr)
        return None, "not capturable (host transport), eager launches"
    return g, "captured (whole step, NCCL calls included)"


def _timed(torch, fn, steps, barrier):
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    e1.synchronize()
    barrier()
    return e0.elapsed_time(e1) / steps


def _first_loss_check(cfg_name, loss, n_gpus):
    path = os.path.join(ROOT, "tests", "golden", "bench_losses.json")
    try:
        ref = json.load(open(path))[cfg_name]["loss"]
    except Exception:
        return {"first_step_loss": loss, "oracle_loss": None, "ok": None, "note": f"no stored oracle loss for {cfg_name}"}
    loss = float(loss)
    rel = float(abs(loss - ref) / abs(ref))
    out = {"first_step_loss": loss, "oracle_loss": ref, "rel_err": rel, "tol": 1e-2, "ok": bool(rel <= 1e-2)}
    if not out["ok"]:
        raise SystemExit(f"[bench] first-step loss {loss} differs from the oracle's {ref} (rel {rel:.2e} > 1e-2)")
    return out


def emulated_halo(a, torch, vm, peaks):
    """N = 1: one rank's block of cfg3's K-way depth split (peer-memory push, or a 1-rank NCCL
    communicator), or of cfg4's 2x2x2 mesh (one-phase NCCL exchange of faces, edges and corners),
    periodic halos, A/B against no exchange (see module docstring)."""
    import numpy as np
    import torch.distributed as dist

    from paper_1909_03108_b200.data import synth_record
    from paper_1909_03108_b200.halo import nccl_comm_ptr
    from paper_1909_03108_b200.step import UNetStep

    # cfg4: one rank's 256^3 block of the 2x2x2 mesh; cfg5: one rank's 256x256x512 block of
    # b=2 x 2x2 spatial (one sample per rank, W unsplit)
    mesh3 = a.emulate_config in ("cfg4", "cfg5")
    K = 8 if mesh3 else a.emulate_split
    c = CONFIGS[a.emulate_config]
    E = c["extent"]
    peer = a.emulate_transport == "peer" and not mesh3  # the peer-memory push covers depth splits
    if not peer and not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    cfg = vm.recipe_for_resolution(E, c["scale"])
    mesh = vm.create_mesh([("one", 1)], backend="threads")
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 1)
    if a.emulate_config == "cfg5":
        loc, nbr6 = (E // 2, E // 2, E), [0, 0, 0, 0, -1, -1]
    elif mesh3:
        loc, nbr6 = (E // 2, E // 2, E // 2), [0] * 6
    else:
        loc, nbr6 = (E // K, E, E), [0, 0, -1, -1, -1, -1]
    st = UNetStep(graph, params, dtype=torch.bfloat16, global_shape=(E, E, E), local_shape=loc)
    if peer:  # vm_halo_depth_push with every neighbour = this rank (wgrad overlaps exchange + dgrad)
        st.use_peer_halo(nbr6=nbr6)
    else:
        comm = nccl_comm_ptr()
        ar = nccl_comm_ptr(dist.new_group(backend="nccl"))
        st.use_nccl(comm, nbr6=nbr6, ar_comm=ar)
    img, lab = synth_record(E, 7, 0)
    blk = (slice(None, 1), slice(0, loc[0]), slice(0, loc[1]), slice(0, loc[2]))
    st.upload(torch.from_numpy(img[None][blk][..., None].copy()), torch.from_numpy(lab[None][blk].copy()))
    for _ in range(2):
        st.step()
    torch.cuda.synchronize()
    # both arms run SGD with lr = 0 (same kernels and bytes): the no-exchange arm computes with
    # wrong margins and, left to train on one sample, diverges within ~10 steps, after which
    # the non-finite values make every later step (of both arms) ~3x slower
    st.lr = 0.0
    fns, graphs = {}, []
    for name, on in (("halo", True), ("nohalo", False)):
        st.has_halo = on
        g, note = _capture(torch, st, not a.no_graph)
        graphs.append(g)
        if g is not None:
            fns[name] = g.replay
        else:
            fns[name] = (lambda on_: (lambda: (setattr(st, "has_halo", on_), st.step())))(on)
    # alternate the two programs (3 rounds, best of each): the A/B is not skewed by drift
    res = {"halo": float("inf"), "nohalo": float("inf")}
    rounds = []
    for _ in range(3):
        for name in ("halo", "nohalo"):
            for _ in range(max(3, a.warmup)):
                fns[name]()
            t = _timed(torch, fns[name], max(5, a.steps), torch.cuda.synchronize)
            rounds.append((name, round(t, 4)))
            res[name] = min(res[name], t)
    del graphs, fns
    st.has_halo = True
    nbytes = st.halo_bytes_per_step()
    # both messages (to the lo and to the hi neighbour) leave through the same NVLink ports:
    # the GPU's egress is 900 GB/s per direction nominal, 770 measured peer copy
    wire_ms = nbytes / (NVLINK_GBS * 1e9) * 1e3
    fwd_bytes = st.halo_bytes_per_step(forward_only=True)
    if peer:
        st.halo.check()
    mesh.shutdown()
    transport = ("peer-memory push (vm_halo_depth_push: one launch per exchange copies the boundary layers into "
                 "the neighbours' margins and signals them; the weight gradient runs concurrently with the "
                 "backward exchange + dgrad)" if peer else
                 "a 1-rank NCCL communicator (pack + NCCL group + unpack per conv)")
    return {
        "share": max(0.0, (res["halo"] - res["nohalo"]) / res["halo"]),
        "method": f"emulated on 1 GPU: rank block {loc[0]}x{loc[1]}x{loc[2]} of "
                  + ({"cfg4": "cfg4's 2x2x2 mesh", "cfg5": "cfg5's b=2 x 2x2 spatial mesh (one sample per rank, "
                      "W unsplit)"}[a.emulate_config] + " (faces, edges and corners in one round of NCCL send/recv, "
                      "vm_halo_slab_fwd26)" if mesh3 else f"cfg3 {K}-way depth split") + ", periodic "
                  f"halos (every neighbour = this rank) through {transport}; "
                  "A/B: (t_step - t_step_nohalo) / t_step, best of 3 alternating rounds, SGD at lr = 0 in both "
                  "arms (same work; keeps the wrong-margin arm from diverging)",
        "transport": "peer" if peer else "nccl",
        "emulated_config": a.emulate_config,
        "rounds_ms": rounds,
        "ms_step": res["halo"], "ms_nohalo": res["nohalo"],
        "bytes_per_step_rank": nbytes,
        "forward_bytes_per_step_rank": fwd_bytes,
        "projected_wire_ms_at_770GBs": wire_ms,
        "projected_share_no_overlap": wire_ms / (res["nohalo"] + wire_ms),
        # forward exchanges sit on the critical path; the backward ones overlap the weight
        # gradients (peer transport): the forward wire time at 770 GB/s on top of the measured step
        "projected_share_fwd_exposed": (fwd_bytes / (NVLINK_GBS * 1e9) * 1e3)
        / (res["halo"] + fwd_bytes / (NVLINK_GBS * 1e9) * 1e3),
        "projected_whole_job_voxels_per_s": K * loc[0] * loc[1] * loc[2] / (res["halo"] * 1e-3),
    }


def scaling_base(a, torch, vm):
    """The 1-GPU point of a strong-scaling series ("cfg3 256^3 b32, 1 GPU
    (scaling base)"): the same network and global volume, unpartitioned, on this process's
    GPU alone, timed like the main run (captured step graph, max(5, steps) steps).  The
    driver's N = 1 run measures cfg2 (BASELINE.json configs[1]); this gives the N > 1 lines
    of cfg3 their own single-GPU denominator."""
    import numpy as np

    from paper_1909_03108_b200.data import synth_record
    from paper_1909_03108_b200.step import UNetStep

    c = CONFIGS[a.config]
    E, B = c["extent"], c["batch"]
    cfg = vm.recipe_for_resolution(E, c["scale"])
    mesh = vm.create_mesh([("one", 1)], backend="threads")
    try:
        graph = vm.build(cfg, mesh, {})
        st = UNetStep(graph, vm.init_params(graph, 1), batch=B, dtype=torch.bfloat16, conv_impl=a.conv)
        recs = [synth_record(E, 7, i) for i in range(B)]
        st.upload(torch.from_numpy(np.stack([r[0] for r in recs])[..., None]),
                  torch.from_numpy(np.stack([r[1] for r in recs])))
        for _ in range(2):
            st.step()
        torch.cuda.synchronize()
        g, note = _capture(torch, st, not a.no_graph)
        fn = g.replay if g is not None else st.step
        for _ in range(max(3, a.warmup)):
            fn()
        ms = _timed(torch, fn, max(5, a.steps), torch.cuda.synchronize)
        out = {"config": f"{a.config} network, {E}^3, global batch {B}, unpartitioned on one GPU (rank 0's)",
               "value": B * E ** 3 / (ms * 1e-3), "unit": "voxels/s", "ms_per_step": ms, "cuda_graph": note,
               "loss": st.loss()[0]}
        del g, fn, st
        return out
    finally:
        mesh.shutdown()
        torch.cuda.empty_cache()


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
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peak_src = load_peaks()
    c = CONFIGS[a.config]
    E, B = c["extent"], c["batch"]
    cfg = vm.recipe_for_resolution(E, c["scale"])
    axes = c["mesh"](world)
    if world > 1:
        mesh = vm.create_mesh(axes)
        layout = c["layout"](world)
    else:
        mesh = vm.create_mesh([("one", 1)], backend="threads")
        layout = {}
    graph = vm.build(cfg, mesh, layout)
    params = vm.init_params(graph, 1)
    ctx = mesh.context(rank) if world > 1 else None
    from paper_1909_03108_b200.training import _blocks

    bdiv = mesh.axis_size(layout["batch"]) if "batch" in layout else 1
    st = UNetStep(graph, params, batch=B // bdiv, ctx=ctx, dtype=torch.bfloat16, conv_impl=a.conv,
                  global_batch=B)
    transport = "none" if world == 1 else "nccl (pack / send-recv group / unpack per phase)"
    if world > 1 and a.halo_transport == "peer" and st.has_halo and max(st.halo.nbr6[2:]) < 0:
        try:  # depth-only split: boundary layers pushed from the conv epilogues over NVLink P2P
            st.use_peer_halo()
            transport = "peer (CUDA-IPC mapped neighbour slabs, pushes fused into the conv epilogues)"
        except Exception as e:  # every rank falls back together (decided collectively)
            print(f"[bench] !!! peer-memory halo unavailable ({e}); NCCL transport", file=sys.stderr, flush=True)
            transport = f"nccl (peer-memory halo failed: {type(e).__name__})"
    recs = [synth_record(E, 7, i) for i in range(B)]
    img = np.stack([r[0] for r in recs])[..., None]
    lab = np.stack([r[1] for r in recs])
    img_h = torch.from_numpy(_blocks(graph, img)[rank]).pin_memory()
    lab_h = torch.from_numpy(_blocks(graph, lab)[rank]).pin_memory()
    del recs, img, lab
    st.upload(img_h, lab_h)
    st.forward()
    torch.cuda.synchronize()
    if transport.startswith("peer"):
        # the peer-memory halo has only run emulated on one GPU before a multi-GPU box: if its
        # first step misses a neighbour's signal or gives the wrong loss on ANY rank, every
        # rank rebuilds the step on the NCCL transport (decided collectively)
        bad = 0
        try:
            st.halo.check()
            _first_loss_check(a.config, st.loss()[0], world)
        except (Exception, SystemExit) as e:
            print(f"[bench] !!! rank {rank}: peer-memory halo failed its first step ({e})", file=sys.stderr, flush=True)
            bad = 1
        flag = torch.tensor([bad], device="cuda", dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if int(flag.item()):
            peer_failed = st  # keep alive: peers may still hold IPC mappings of its slabs
            st = UNetStep(graph, params, batch=B // bdiv, ctx=ctx, dtype=torch.bfloat16, conv_impl=a.conv,
                          global_batch=B)
            transport = "nccl (peer-memory halo failed its first step)"
            st.upload(img_h, lab_h)
            st.forward()
            torch.cuda.synchronize()
            del peer_failed
    parity = _first_loss_check(a.config, st.loss()[0], world)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(2):  # eager warm-up (first-touch of every kernel and plan)
        st.step()
    torch.cuda.synchronize()
    l0 = _lib.load().vm_launch_count()
    st.step()
    torch.cuda.synchronize()
    launches_per_step = _lib.load().vm_launch_count() - l0
    graph_obj, graph_note = _capture(torch, st, not a.no_graph)
    one = graph_obj.replay if graph_obj is not None else st.step
    for _ in range(a.warmup):
        one()
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs
    with ClockSampler(local) as clk:
        ms = max_over_ranks(_timed(torch, one, a.steps, barrier))
    voxels = B * E ** 3  # the whole job's voxels per step
    value = voxels / (ms * 1e-3)

    # ---- end to end through the public API: host buffers, H2D + D2H inside the timed region
    st.train_loop_host([(img_h, lab_h)] * max(a.warmup, 1), replay=one)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    losses = st.train_loop_host([(img_h, lab_h)] * a.steps, replay=one)
    f1.record()
    f1.synchronize()
    barrier()
    ms_e2e = max_over_ranks(f0.elapsed_time(f1) / a.steps)
    h2d = img_h.numel() * img_h.element_size() + lab_h.numel() * lab_h.element_size()
    d2h = st.stats.numel() * 4 + 4

    # ---- halo share
    if world > 1:
        # A/B of the same step with the exchange on / off, both arms at lr = 0 (same kernels and
        # bytes: the wrong-margin arm would otherwise diverge and its non-finite values slow
        # every later step), alternating 3 rounds, best of each, max over ranks
        st.lr = 0.0
        arms = {}
        for name, on in (("halo", True), ("nohalo", False)):
            st.has_halo = on
            g2, _ = _capture(torch, st, not a.no_graph)
            arms[name] = (g2, g2.replay if g2 is not None else
                          (lambda on_: (lambda: (setattr(st, "has_halo", on_), st.step())))(on))
        best = {"halo": float("inf"), "nohalo": float("inf")}
        for _ in range(3):
            for name in ("halo", "nohalo"):
                for _ in range(a.warmup):
                    arms[name][1]()
                best[name] = min(best[name], max_over_ranks(_timed(torch, arms[name][1], a.steps, barrier)))
        del arms
        st.has_halo = True
        ms_ab, ms_nohalo = best["halo"], best["nohalo"]
        nbytes = st.halo_bytes_per_step()
        halo = {"share": max(0.0, (ms_ab - ms_nohalo) / ms_ab), "method": "A/B: (t_step - t_step_nohalo) / t_step, "
                "no-halo = same kernels with the exchange off (margins stale: timing only), both arms at lr = 0, "
                "3 alternating rounds, best of each, max over ranks",
                "transport": transport, "ms_step_ab": ms_ab,
                "ms_nohalo": ms_nohalo, "bytes_per_step_rank": nbytes,
                "exchange_byte_count_per_step": halo_formula_bytes(vm, graph, mesh, layout, B),
                "nvlink_gbs_achieved_if_exposed": nbytes / max(ms_ab - ms_nohalo, 1e-6) / 1e6}
        if transport.startswith("peer"):
            try:  # a neighbour signal missed during the timed steps would have left stale margins
                st.halo.check()
            except Exception as e:  # noqa: BLE001
                halo["error"] = str(e)
    elif not a.no_emulate:
        try:
            halo = emulated_halo(a, torch, vm, peaks)
        except Exception as e:  # pragma: no cover
            halo = {"share": None, "method": f"emulation failed: {type(e).__name__}: {e}"}
        if a.emulate_config == "cfg3" and not a.no_emulate_cfg4:
            # the 3-D meshes too: one rank block of cfg4 (2x2x2) and of cfg5 (b=2 x 2x2), faces +
            # edges + corners through the one-phase NCCL exchange (vm_halo_slab_fwd26)
            import copy

            for name, key in (("cfg4", "cfg4_2x2x2"), ("cfg5", "cfg5_b2x2x2")):
                b = copy.copy(a)
                b.emulate_config = name
                try:
                    halo[key] = emulated_halo(b, torch, vm, peaks)
                except Exception as e:  # pragma: no cover
                    halo[key] = {"share": None, "method": f"emulation failed: {type(e).__name__}: {e}"}
                torch.cuda.empty_cache()
    else:
        halo = {"share": 0.0, "method": "one GPU, no partitioning"}

    # ---- per-kernel timing for the roofline (each launch replayed alone as a CUDA graph)
    prof = st.profile_kernels(reps=5)
    classes = {}
    for row in prof:
        cc = classes.setdefault(row["kind"], {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0, "att_ms": 0.0})
        cc["ms"] += row["ms"]
        cc["flops"] += row["flops"]
        cc["bytes"] += row["bytes"]
        cc["launches"] += 1
        # per-launch roofline time: the slower of its FLOPs at the tensor peak and its
        # algorithmic bytes at the HBM peak (thin layers are memory-bound: 16->16 wgrad at
        # 128^3 moves 134 MB for 29 GFLOP, 20.5 us at 6.55 TB/s against 17.5 us at 1658 TF/s)
        cc["att_ms"] += max(row["flops"] / (peaks["bf16_tflops"] * 1e9), row["bytes"] / (peaks["hbm_gbs"] * 1e6))
    dom_kind = max(classes, key=lambda k: classes[k]["ms"])
    dom = classes[dom_kind]
    step_kernel_ms = sum(cc["ms"] for cc in classes.values())
    traffic, traffic_src = load_traffic(dom_kind, a.config)
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
                 "traffic_source": traffic_src,
                 "attainable_frac": dom["att_ms"] / dom["ms"],
                 "attainable_note": "sum over launches of max(flops / tensor peak, algorithmic bytes / HBM peak) "
                                    "divided by the measured time (each launch against its own roofline)"})
    conv_flops_rank = sum(cc["flops"] for k, cc in classes.items() if k.startswith("conv"))
    conv_ms = sum(cc["ms"] for k, cc in classes.items() if k.startswith("conv"))
    act_gb = torch.cuda.max_memory_allocated() / 1e9
    if a.layer_csv and rank == 0:
        with open(a.layer_csv, "w") as f:
            f.write("layer,kind,ms,flops,bytes,tflops,gbs\n")
            for r in prof:
                f.write(f"{r['layer']},{r['kind']},{r['ms']:.4f},{r['flops']:.0f},{r['bytes']:.0f},"
                        f"{r['flops'] / max(r['ms'], 1e-9) / 1e9:.1f},{r['bytes'] / max(r['ms'], 1e-9) / 1e6:.1f}\n")

    base = None
    if a.config == "cfg3" and (a.scaling_base == "on" or (a.scaling_base == "auto" and world > 1)):
        if rank == 0:  # the other ranks wait at the barrier below (outside every timed region)
            try:
                base = scaling_base(a, torch, vm)
            except Exception as e:  # noqa: BLE001
                base = {"value": None, "error": f"{type(e).__name__}: {e}"}
        if world > 1:
            dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not a.no_cpu:
        try:
            v, per, cores, sample, _ = cpu_sample(a.config, 60.0, max_steps=1)
            cpu = {"value": v, "unit": "voxels/s", "cores": cores, "kind": "port", "sample": sample}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "voxels/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}
    wl = workload(a)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "voxels/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (data_io.synthesize_record distribution, SeedSequence([7, i]) for sample i)",
        "config": wl,
        "run": {"conv": a.conv, "cuda_graph": graph_note, "memory_gb_peak": round(act_gb, 1),
                "l2": f"working set {act_gb:.1f} GB >> 126 MB L2; no flush needed",
                "conv_tflop_per_step_rank": conv_flops_rank / 1e12,
                "transport": transport + ("; collectives: NCCL via C ABI (vm_allreduce_f32)" if world > 1 else "")},
        "parity": parity,
        "e2e": {"value": voxels / (ms_e2e * 1e-3), "unit": "voxels/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e, "loss": losses[-1][0],
                "path": "UNetStep.train_loop_host: per step pinned H2D (prefetched one step ahead on a copy "
                        "stream) -> slab kernels -> step graph -> async D2H of the loss statistics"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * a.steps,
        "halo": halo,
        **({"scaling_base": base} if base is not None else {}),
        "kernel_ms_per_step": {k: round(cc["ms"], 4) for k, cc in classes.items()},
        "roofline_by_kind": {
            k: ({"bound": "tensor", "tflops": round(cc["flops"] / (cc["ms"] * 1e-3) / 1e12, 1),
                 "frac": round(cc["flops"] / (cc["ms"] * 1e-3) / 1e12 / peaks["bf16_tflops"], 3),
                 "attainable_frac": round(cc["att_ms"] / cc["ms"], 3)}
                if cc["flops"] > 0 and k.startswith("conv") else
                {"bound": "hbm", "gbs": round(cc["bytes"] / (cc["ms"] * 1e-3) / 1e9, 0),
                 "frac": round(cc["bytes"] / (cc["ms"] * 1e-3) / 1e9 / peaks["hbm_gbs"], 3)})
            for k, cc in classes.items() if cc["ms"] > 0},
        "conv_tflops_effective": conv_flops_rank / (conv_ms * 1e-3) / 1e12 if conv_ms else None,
    }
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def halo_formula_bytes(vm, graph, mesh, layout, B):
    """exchange_byte_count (halo.py:197-229) of every k = 3 conv input, fwd + bwd (the first
    conv has no backward exchange), bf16, summed over all ranks."""
    tot = 0
    halo = vm.HaloSpec.for_kernel(3)
    lay = vm.Layout(layout)
    for n in graph.conv_nodes:
        if n.k != 3:
            continue
        e = graph.level_extents[n.id]
        spec = vm.TensorSpec((("batch", B), ("x", e), ("y", e), ("z", e), ("c", n.c_in)), "u8")
        one = vm.exchange_byte_count(spec, lay, mesh, halo) * 2  # bf16 = 2 bytes per element
        tot += one * (1 if n.inputs[0] == "input" else 2)
    return tot


def main():
    a = args_parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
