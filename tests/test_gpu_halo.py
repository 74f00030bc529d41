"""GPU halo exchange (threads mesh on one device) vs the oracle protocol: bit-exact."""

import numpy as np
import pytest

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O

pytestmark = pytest.mark.gpu


def _spec(b, e, c, dtype="f32"):
    return vm.TensorSpec((("batch", b), ("x", e), ("y", e), ("z", e), ("c", c)), dtype)


def test_1d_exchange_hand_checked():
    with vm.create_mesh([("ax", 2)]) as mesh:
        spec = vm.TensorSpec((("x", 8),))
        st = vm.shard(np.arange(8, dtype=np.float32), spec, vm.Layout({"x": "ax"}), mesh)
        padded = vm.halo_exchange(st, vm.HaloSpec((("x", 1, 1),)))
        mesh.synchronize()
        assert np.array_equal(padded[0].data.cpu().numpy(), [0, 0, 1, 2, 3, 4])
        assert np.array_equal(padded[1].data.cpu().numpy(), [3, 4, 5, 6, 7, 0])
        assert padded[0].faces[("x", "lo")] == "zero"
        assert padded[0].faces[("x", "hi")] == "neighbor"


@pytest.mark.parametrize("dtype", ["f32", "f64", "u8"])
def test_222_padded_blocks_match_oracle_bitwise(dtype):
    axes = [("mx", 2), ("my", 2), ("mz", 2)]
    lay = {"x": "mx", "y": "my", "z": "mz"}
    rng = np.random.default_rng(1)
    spec = _spec(2, 8, 3, dtype)
    x = (rng.standard_normal(spec.shape) * 50).astype(spec.dtype)
    halo = vm.HaloSpec.for_kernel(3)
    with vm.create_mesh(axes) as mesh:
        layout = vm.Layout(lay)
        st = vm.shard(x, spec, layout, mesh)
        b0 = mesh.run(lambda ctx: ctx.counters["p2p_bytes"])
        padded = vm.halo_exchange(st, halo)
        b1 = mesh.run(lambda ctx: ctx.counters["p2p_bytes"])
        mesh.synchronize()
        dims = spec.dims
        ref, nbytes = O.halo_exchange_blocks(
            O.shard_blocks(x, dims, lay, axes), dims, lay, axes, {d: (1, 1) for d in "xyz"}
        )
        for r in range(mesh.worker_count):
            assert np.array_equal(padded[r].data.cpu().numpy(), ref[r])
        assert sum(b1) - sum(b0) == vm.exchange_byte_count(spec, layout, mesh, halo) == nbytes


def test_backward_matches_oracle_adjoint_bitwise():
    axes = [("mx", 2), ("my", 2), ("mz", 2)]
    lay = {"x": "mx", "y": "my", "z": "mz"}
    rng = np.random.default_rng(5)
    spec = _spec(1, 8, 2)
    halo = vm.HaloSpec((("x", 1, 1), ("y", 2, 2), ("z", 1, 1)))
    with vm.create_mesh(axes) as mesh:
        layout = vm.Layout(lay)
        ys = [rng.standard_normal((1, 6, 8, 6, 2)).astype(np.float32) for _ in range(8)]
        import torch

        dev = [torch.from_numpy(y).to(mesh.device_of(r)) for r, y in enumerate(ys)]
        back = vm.halo_exchange_backward(dev, spec, layout, mesh, halo)
        got = vm.gather(back)
        ref_blocks = O.halo_exchange_backward_blocks(ys, spec.dims, lay, axes, {"x": (1, 1), "y": (2, 2), "z": (1, 1)})
        ref = O.gather_blocks(ref_blocks, spec.dims, lay, axes, np.float32)
        assert np.array_equal(got, ref)


def test_margin_exceeding_local_extent_suggests_fix():
    with vm.create_mesh([("mx", 2)]) as mesh:
        spec = _spec(1, 8, 1)
        st = vm.shard(np.zeros(spec.shape, np.float32), spec, vm.Layout({"x": "mx"}), mesh)
        with pytest.raises(vm.WorkerFailed, match="smaller mesh axis or a larger volume"):
            vm.halo_exchange(st, vm.HaloSpec((("x", 5, 5),)))
