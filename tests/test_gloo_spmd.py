"""The spmd transport (one process per rank, torch.distributed) exercised on CPU with
gloo at world size 2: topology, all-reduce, gather, and the halo protocol's grouped
send/recv (batch_isend_irecv) vs the oracle, bitwise.  On the GPU box the same code
runs over NCCL with the CUDA pack kernels."""

import os
import socket
import sys
import traceback

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    try:
        sys.path.insert(0, ROOT)
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1909_03108_b200 as vm
        from oracle import voxmesh_oracle as O
        from paper_1909_03108_b200.halo import dim_axes, exchange_backward_local, exchange_local
        from tests.helpers import TorchPacker

        res = {}
        mesh = vm.create_mesh([("mx", world)], devices=["cpu"])
        assert mesh.backend == "spmd" and mesh.local_ranks == [rank]
        ctx = mesh.context(rank)
        red = mesh.run(lambda c: c.all_reduce_sum(np.array([rank + 1.0, 10.0 * rank])))[rank]
        res["allreduce"] = red.tolist()
        t = mesh.run(lambda c: c.all_reduce_sum(torch.tensor([float(rank)])))[rank]
        res["allreduce_t"] = float(t[0])

        spec = vm.TensorSpec((("batch", 1), ("x", 8), ("y", 6), ("z", 4), ("c", 3)))
        layout = vm.Layout({"x": "mx"})
        x = np.random.default_rng(11).standard_normal(spec.shape).astype(np.float32)
        st = vm.shard(x, spec, layout, mesh)
        res["gather_ok"] = bool(np.array_equal(vm.gather(st), x))
        dims = dim_axes(spec, layout)
        halo = vm.HaloSpec.for_kernel(3)
        pb = mesh.run(lambda c, b: exchange_local(c, dims, halo, "halo", True, b, packer=TorchPacker()),
                      per_worker=(st.blocks,))[rank]
        ref, _ = O.halo_exchange_blocks(O.shard_blocks(x, spec.dims, {"x": "mx"}, [("mx", world)]), spec.dims,
                                        {"x": "mx"}, [("mx", world)], {d: (1, 1) for d in "xyz"})
        res["halo_ok"] = bool(np.array_equal(pb.data.numpy(), ref[rank]))
        res["bytes"] = ctx.counters["p2p_bytes"]
        rng = np.random.default_rng(99)
        ys = [rng.standard_normal(r.shape).astype(np.float32) for r in ref]
        back = mesh.run(lambda c, g: exchange_backward_local(c, dims, halo, "halo-bwd", True, g, packer=TorchPacker()),
                        per_worker=([torch.from_numpy(y) for y in ys],))[rank]
        rback = O.halo_exchange_backward_blocks(ys, spec.dims, {"x": "mx"}, [("mx", world)], {d: (1, 1) for d in "xyz"})
        res["adjoint_ok"] = bool(np.array_equal(back.numpy(), rback[rank]))
        dist.destroy_process_group()
        out.put((rank, res, None))
    except Exception:  # pragma: no cover - surfaced to the parent
        out.put((rank, None, traceback.format_exc()))


def test_spmd_transport_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=240)
        assert err is None, err
        results[rank] = res
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert results[r]["allreduce"] == [3.0, 10.0]
        assert results[r]["allreduce_t"] == 1.0
        assert results[r]["gather_ok"] and results[r]["halo_ok"] and results[r]["adjoint_ok"]
    # each rank sends one (6+2)x(4+2)... face: total equals the analytic formula
    import paper_1909_03108_b200 as vm

    class _M:
        axes = [type("A", (), {"name": "mx", "size": 2})()]
        axis_index = {"mx": 0}
        coords = [(0,), (1,)]

        @staticmethod
        def axis_size(a):
            return 2

    spec = vm.TensorSpec((("batch", 1), ("x", 8), ("y", 6), ("z", 4), ("c", 3)))
    assert results[0]["bytes"] + results[1]["bytes"] == vm.exchange_byte_count(
        spec, vm.Layout({"x": "mx"}), _M(), vm.HaloSpec.for_kernel(3))
