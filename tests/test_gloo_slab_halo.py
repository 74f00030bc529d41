"""The U-Net step's slab halo (halo.SlabHalo: the 3-phase protocol on channel-blocked padded
slabs, batched per phase) over the spmd transport on CPU: gloo, one process per rank, world
sizes 2 (depth split) and 4 (2 x 2), against the oracle's halo protocol (halo.py:109-155),
bitwise; the bytes sent equal exchange_byte_count; zero() clears exactly the margins that
came from neighbours.  On the GPU box the same class drives the CUDA pack/unpack kernels, or
the whole exchange through the NCCL C ABI."""

import os
import socket
import sys
import traceback

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, axes, lay, out):
    try:
        sys.path.insert(0, ROOT)
        import torch
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1909_03108_b200 as vm
        from oracle import voxmesh_oracle as O
        from paper_1909_03108_b200.halo import SlabHalo, TorchSlabKernels
        from paper_1909_03108_b200.step import Slab

        mesh = vm.create_mesh(axes, devices=["cpu"])
        ctx = mesh.context(rank)
        B, E, C = 2, 8, 11  # two channel groups, the second one partly padding
        dims = (("batch", B), ("x", E), ("y", E), ("z", E), ("c", C))
        x = np.random.default_rng(5).standard_normal([e for _, e in dims]).astype(np.float32)
        blocks = O.shard_blocks(x, dims, lay, axes)
        ref, _ = O.halo_exchange_blocks(blocks, dims, lay, axes, {d: (1, 1) for d in "xyz"})
        blk = blocks[rank]
        _, D, H, W, _ = blk.shape
        s = Slab(B, C, D, H, W, torch.float32, "cpu")
        v = TorchSlabKernels.view(s)
        dense = torch.zeros(B, D, H, W, s.CG * 8)
        dense[..., :C] = torch.from_numpy(blk)
        v[:, :, 1:-1, 1:-1, 1:-1, :] = dense.reshape(B, D, H, W, s.CG, 8).permute(0, 4, 1, 2, 3, 5)
        nbr6 = []
        for d in ("x", "y", "z"):
            a = lay.get(d)
            nbr6 += [-1, -1] if a is None else [ctx.neighbor(a, -1) if ctx.neighbor(a, -1) is not None else -1,
                                                ctx.neighbor(a, +1) if ctx.neighbor(a, +1) is not None else -1]
        halo = SlabHalo(nbr6, ctx=ctx, kernels=TorchSlabKernels())
        halo.forward(s)
        got = v.permute(0, 2, 3, 4, 1, 5).reshape(B, D + 2, H + 2, W + 2, s.CG * 8)[..., :C].numpy()
        res = {"halo_ok": bool(np.array_equal(got, ref[rank])), "bytes": ctx.counters["p2p_bytes"]}
        halo.zero(s)
        z = v.permute(0, 2, 3, 4, 1, 5).reshape(B, D + 2, H + 2, W + 2, s.CG * 8)[..., :C].numpy()
        ok = np.array_equal(z[:, 1:-1, 1:-1, 1:-1], blk)
        for a in range(3):
            for side, pos in ((0, 0), (1, -1)):
                idx = [slice(None)] * 5
                idx[1 + a] = pos
                face = z[tuple(idx)]
                if nbr6[2 * a + side] >= 0:
                    ok &= not np.any(face)
        res["zero_ok"] = bool(ok)
        dist.destroy_process_group()
        out.put((rank, res, None))
    except Exception:  # pragma: no cover - surfaced to the parent
        out.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("axes,lay", [
    ([("mx", 2)], {"x": "mx"}),
    ([("mx", 2), ("my", 2)], {"x": "mx", "y": "my"}),
])
def test_slab_halo_gloo_matches_oracle(axes, lay):
    world = int(np.prod([s for _, s in axes]))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, axes, lay, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=300)
        assert err is None, err
        results[rank] = res
    for p in procs:
        p.join(timeout=60)
    sys.path.insert(0, ROOT)
    import paper_1909_03108_b200 as vm

    class _M:
        def __init__(self):
            self.axes = [type("A", (), {"name": n, "size": s})() for n, s in axes]
            self.axis_index = {n: i for i, (n, _) in enumerate(axes)}
            import itertools

            self.coords = list(itertools.product(*[range(s) for _, s in axes]))

        def axis_size(self, a):
            return dict(axes)[a]

    spec = vm.TensorSpec((("batch", 2), ("x", 8), ("y", 8), ("z", 8), ("c", 16)))  # CG * 8 channels travel
    want = vm.exchange_byte_count(spec, vm.Layout(lay), _M(), vm.HaloSpec.for_kernel(3))
    assert sum(r["bytes"] for r in results.values()) == want
    for r in range(world):
        assert results[r]["halo_ok"] and results[r]["zero_ok"], (r, results[r])
