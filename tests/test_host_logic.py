"""Host-side logic of the product on CPU: builder / init vs the reference's golden
vectors, partitioner, mesh topology + collectives (threads transport), the halo
protocol plan driven through the mesh with a test packer, ABI exports."""

import math
import os
import re

import numpy as np
import pytest
import torch

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.data import synth_record
from paper_1909_03108_b200.halo import exchange_backward_local, exchange_local
from tests.helpers import TorchPacker

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "voxmesh_golden.npz"))


# ---------------------------------------------------------------- builder / init
def test_recipes_match_reference():
    for row in G["recipes"]:
        ext, sc = int(row[0]), float(row[1])
        assert vm.recipe_for_resolution(ext, sc).encoder_filters == tuple(int(v) for v in row[2:] if v)
    # test_unet.py:17-30 ladders
    assert vm.recipe_for_resolution(64).encoder_filters == (256, 512, 1024)
    assert vm.recipe_for_resolution(128).encoder_filters == (128, 256, 512, 1024)


@pytest.mark.parametrize("name,ext,sc", [("cfg2", 128, 0.125), ("cfg4", 512, 1.0)])
def test_graph_matches_reference(name, ext, sc):
    with vm.create_mesh([("one", 1)]) as mesh:
        g = vm.build(vm.recipe_for_resolution(ext, sc), mesh, {})
    assert [n.id for n in g.nodes] == list(G[f"graph_{name}_ids"])
    assert [n.op for n in g.nodes] == list(G[f"graph_{name}_ops"])
    assert [n.c_in for n in g.nodes] == list(G[f"graph_{name}_cin"])
    assert [n.c_out for n in g.nodes] == list(G[f"graph_{name}_cout"])
    assert g.param_count == int(G[f"graph_{name}_params"])
    assert g.receptive_field() == int(G[f"graph_{name}_rf"])


def test_conv_flops_of_baseline_configs():
    # cfg2 1.445 TFLOP, cfg4 401.66 TFLOP per step (fwd + dgrad w/o first conv + wgrad)
    with vm.create_mesh([("one", 1)]) as mesh:
        g2 = vm.build(vm.recipe_for_resolution(128, 0.125), mesh, {})
        g4 = vm.build(vm.recipe_for_resolution(512, 1.0), mesh, {})
    assert abs(g2.conv_flops() / 1e12 - 1.445) < 0.001
    assert abs(g4.conv_flops() / 1e12 - 401.66) < 0.01


def test_param_count_hand_value_and_receptive_field():
    with vm.create_mesh([("one", 1)]) as mesh:
        g = vm.build(vm.UNetConfig(8, (2, 4), convs_per_block=1), mesh, {})
        assert g.param_count == (27 * 2 + 2) + (27 * 8 + 4) + (27 * 12 + 2) + (2 * 3 + 3)
        g = vm.build(vm.UNetConfig(32, (8, 16), convs_per_block=4), mesh, {})
        assert g.receptive_field() == 33


def test_init_params_bitwise_reference():
    with vm.create_mesh([("one", 1)]) as mesh:
        g = vm.build(vm.UNetConfig(8, (2, 4), convs_per_block=2), mesh, {})
    p = vm.init_params(g, 5)
    for nid, d in p.items():
        assert np.array_equal(d["kernel"], G[f"net_p_{nid}_kernel"])
        assert not d["bias"].any()


def test_build_errors_use_reference_wording():
    with vm.create_mesh([("mx", 2), ("my", 2)]) as mesh:
        with pytest.raises(vm.GraphBuildError, match="not used by the layout"):
            vm.build(vm.UNetConfig(8, (2, 4)), mesh, {"x": "mx"})
        with pytest.raises(vm.GraphBuildError, match="pooling needs an even local extent"):
            vm.build(vm.UNetConfig(4, (2, 4, 8)), mesh, {"x": "mx", "y": "my"})
    with vm.create_mesh([("mx", 4)]) as mesh:
        with pytest.raises(vm.GraphBuildError, match="smaller mesh axis or a larger volume"):
            vm.build(vm.UNetConfig(4, (2,), kernel=5), mesh, {"x": "mx"})
    with pytest.raises(vm.GraphBuildError, match="double"):
        vm.UNetConfig(8, (2, 5))
    cfg = vm.UNetConfig(32, (8, 16), convs_per_block=3)
    assert vm.UNetConfig.from_kv(cfg.to_kv()) == cfg


def test_synthetic_record_bitwise_reference():
    img, lab = synth_record(16, 7, 0)
    assert np.array_equal(img, G["synth16_image"]) and np.array_equal(lab, G["synth16_labels"])
    img2, lab2 = O.record_for(24, 3)
    a, b = synth_record(24, 7, 3)
    assert np.array_equal(a, img2) and np.array_equal(b, lab2)


# ---------------------------------------------------------------- partitioner
def test_spec_and_layout_validation():
    with pytest.raises(vm.ShardingError):
        vm.TensorSpec((("x", 4), ("x", 4)))
    with pytest.raises(vm.ShardingError):
        vm.TensorSpec((("x", 4),), "f16")
    with pytest.raises(vm.ShardingError, match="channel dimension"):
        vm.Layout({"c": "mx"})
    with pytest.raises(vm.ShardingError, match="one mesh axis"):
        vm.Layout({"x": "mx", "y": "mx"})
    with vm.create_mesh([("ax", 3)]) as mesh:
        with pytest.raises(vm.ShardingError, match=r"'x' extent 8.*'ax' of size 3"):
            vm.shard(np.zeros(8, np.float32), vm.TensorSpec((("x", 8),)), vm.Layout({"x": "ax"}), mesh)


@pytest.mark.parametrize("dtype", ["f32", "f64", "u8", "bf16"])
def test_shard_gather_roundtrip_bitwise(dtype):
    rng = np.random.default_rng(3)
    spec = vm.TensorSpec((("batch", 2), ("x", 8), ("y", 4), ("z", 6), ("c", 3)), dtype)
    x = (rng.standard_normal(spec.shape) * 40).astype(np.float32 if dtype == "bf16" else spec.dtype)
    if dtype == "bf16":
        x = O.bf16_round(x)
    with vm.create_mesh([("b", 2), ("mx", 2), ("my", 2)]) as mesh:
        st = vm.shard(x, spec, vm.Layout({"batch": "b", "x": "mx", "y": "my"}), mesh)
        assert st.local_shape == (1, 4, 2, 6, 3)
        assert np.array_equal(vm.gather(st), x)
        assert np.array_equal(st.blocks[0].float().numpy() if dtype == "bf16" else st.blocks[0].numpy(),
                              x[0:1, 0:4, 0:2])


# ---------------------------------------------------------------- mesh (threads transport)
def test_mesh_topology_and_groups():
    with vm.create_mesh([("mx", 2), ("my", 3)]) as mesh:
        assert mesh.coords[4] == (1, 1) and mesh.rank_of[(0, 2)] == 2
        ctx = mesh.context(4)
        assert ctx.neighbor("mx", -1) == 1 and ctx.neighbor("mx", +1) is None
        assert ctx.neighbor("my", +1) == 5
        assert ctx.group("my") == [3, 4, 5] and ctx.group() == list(range(6))
        assert mesh.describe() == "mx=2,my=3"
    with pytest.raises(vm.errors.MeshConfigError):
        vm.create_mesh([("a", 2), ("a", 2)])


def test_all_reduce_sum_coordinate_order_and_subgroups():
    with vm.create_mesh([("mx", 2), ("my", 2)]) as mesh:
        res = mesh.run(lambda ctx: ctx.all_reduce_sum(np.array([ctx.rank + 1.0, 2.0 * ctx.rank])))
        assert all(np.array_equal(r, [10.0, 12.0]) for r in res)
        sub = mesh.run(lambda ctx: ctx.all_reduce_sum(np.array([float(ctx.rank)]), axes="my"))
        assert [float(s[0]) for s in sub] == [1.0, 1.0, 5.0, 5.0]
        with pytest.raises(vm.WorkerFailed):
            mesh.run(lambda ctx: ctx.all_reduce_sum(np.zeros(ctx.rank + 1)))


def test_worker_failure_poisons_mesh():
    with vm.create_mesh([("mx", 2)]) as mesh:
        def boom(ctx):
            if ctx.rank == 1:
                raise ValueError("boom")
            return ctx.recv(1, "never")

        with pytest.raises(vm.WorkerFailed, match="boom"):
            mesh.run(boom)
        with pytest.raises(vm.errors.ProtocolError, match="broken"):
            mesh.run(lambda ctx: None)


# ---------------------------------------------------------------- halo protocol (plan + transport)
PK = TorchPacker()


def _exchange(mesh, x, spec, layout, halo):
    dims = vm.halo.dim_axes(spec, layout)
    st = vm.shard(x, spec, layout, mesh)
    return mesh.run(lambda ctx, blk: exchange_local(ctx, dims, halo, "halo", True, blk, packer=PK), per_worker=(st.blocks,))


@pytest.mark.parametrize("axes,lay", [
    ([("mx", 2), ("my", 2), ("mz", 2)], {"x": "mx", "y": "my", "z": "mz"}),
    ([("mx", 4)], {"x": "mx"}),
    ([("b", 2), ("mx", 2), ("my", 2)], {"batch": "b", "x": "mx", "y": "my"}),
])
def test_halo_protocol_matches_oracle_bitwise(axes, lay):
    spec = vm.TensorSpec((("batch", 2), ("x", 8), ("y", 8), ("z", 4), ("c", 3)))
    x = np.random.default_rng(7).standard_normal(spec.shape).astype(np.float32)
    with vm.create_mesh(axes) as mesh:
        got = _exchange(mesh, x, spec, vm.Layout(lay), vm.HaloSpec.for_kernel(3))
        ref, nbytes = O.halo_exchange_blocks(O.shard_blocks(x, spec.dims, lay, axes), spec.dims, lay, axes,
                                             {d: (1, 1) for d in "xyz"})
        for r in range(mesh.worker_count):
            assert np.array_equal(got[r].data.numpy(), ref[r])
        sent = sum(mesh.run(lambda ctx: ctx.counters["p2p_bytes"]))
        assert sent == vm.exchange_byte_count(spec, vm.Layout(lay), mesh, vm.HaloSpec.for_kernel(3)) == nbytes


def test_halo_adjoint_protocol_matches_oracle_bitwise():
    axes, lay = [("mx", 2), ("my", 2), ("mz", 2)], {"x": "mx", "y": "my", "z": "mz"}
    spec = vm.TensorSpec((("batch", 1), ("x", 8), ("y", 8), ("z", 8), ("c", 2)))
    halo = vm.HaloSpec((("x", 1, 1), ("y", 2, 2), ("z", 1, 1)))
    rng = np.random.default_rng(5)
    ys = [rng.standard_normal((1, 6, 8, 6, 2)).astype(np.float32) for _ in range(8)]
    with vm.create_mesh(axes) as mesh:
        dims = vm.halo.dim_axes(spec, vm.Layout(lay))
        got = mesh.run(lambda ctx, g: exchange_backward_local(ctx, dims, halo, "halo-bwd", True, g, packer=PK),
                       per_worker=([torch.from_numpy(y) for y in ys],))
        ref = O.halo_exchange_backward_blocks(ys, spec.dims, lay, axes, {"x": (1, 1), "y": (2, 2), "z": (1, 1)})
        for r in range(8):
            assert np.array_equal(got[r].numpy(), ref[r])


def test_halo_margin_too_large_message():
    with vm.create_mesh([("mx", 2)]) as mesh:
        spec = vm.TensorSpec((("batch", 1), ("x", 8), ("y", 8), ("z", 8), ("c", 1)))
        with pytest.raises(vm.WorkerFailed, match="smaller mesh axis or a larger volume"):
            _exchange(mesh, np.zeros(spec.shape, np.float32), spec, vm.Layout({"x": "mx"}), vm.HaloSpec((("x", 5, 5),)))


def test_halospec_validation():
    with pytest.raises(vm.HaloError):
        vm.HaloSpec.for_kernel(4)
    with pytest.raises(vm.HaloError):
        vm.HaloSpec((("batch", 1, 1),))
    assert vm.HaloSpec.for_kernel(5).margin("x") == (2, 2)


# ---------------------------------------------------------------- C ABI
def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "vm_api.h")).read()
    declared = set(re.findall(r"\b(vm_[a-z0-9_]+)\s*\(", header))
    lib = _lib.load()
    missing = sorted(n for n in declared if getattr(lib, n, None) is None)
    assert not missing, missing
    assert lib.vm_version() >= 1
    assert lib.vm_error_string(-5) == b"halo margin exceeds local extent"


def test_no_cpu_fallback_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(vm.VoxmeshError, match="no CPU fallback"):
        _lib.stream_ptr()


def test_conv_params_validation():
    k = np.zeros((3, 3, 3, 2, 4), np.float32)
    vm.ConvParams(k, np.zeros(4, np.float32))
    with pytest.raises(vm.HaloError):
        vm.ConvParams(np.zeros((2, 2, 2, 2, 4), np.float32), np.zeros(4, np.float32))
    with pytest.raises(vm.VoxmeshError):
        vm.ConvParams(k, np.zeros(3, np.float32))
    with pytest.raises(vm.VoxmeshError):
        vm.ConvParams(np.full((3, 3, 3, 2, 4), np.nan, np.float32), np.zeros(4, np.float32))


def test_augment_config_and_quantize_host_side():
    # SynthConfig validation (augment.py:40-45) and the 1/256 delta snap (:48-50)
    from paper_1909_03108_b200 import augment as A
    from paper_1909_03108_b200.errors import AugmentError
    with pytest.raises(AugmentError):
        A.SynthConfig(n_tumors=(0, 2))
    with pytest.raises(AugmentError):
        A.SynthConfig(n_tumors=(3, 2))
    with pytest.raises(AugmentError):
        A.SynthConfig(radius_range=(0.5, 2.0))
    assert A.quantize_delta(0.3) == float(np.float32(round(0.3 * 256) / 256))
    assert A.with_seed(A.SynthConfig(), 7).seed == 7


def test_one_phase_directions_rebuild_the_global_padding_on_a_2x2x2_mesh():
    """nbr26_of / directions26 (the neighbour table of vm_halo_slab_fwd26): boxes sent in
    direction k and received from the neighbour at offset opp(k) = 25 - k, in the C call's
    order, give every rank of a 2x2x2 mesh the slice of the globally zero-padded volume
    (faces, edges and corners; halo.py:109-155's result without its 3 hops)."""
    import itertools

    from paper_1909_03108_b200.halo import directions26, nbr26_of

    n = (3, 4, 5)
    g = np.random.default_rng(0).standard_normal((2 * n[0], 2 * n[1], 2 * n[2]))
    gp = np.pad(g, 1)
    coords = list(itertools.product(range(2), repeat=3))
    rank_of = {c: r for r, c in enumerate(coords)}
    dirs = directions26()
    assert all(tuple(-v for v in dirs[k]) == dirs[25 - k] for k in range(26))
    blocks, n26 = [], []
    for c in coords:
        b = np.zeros(tuple(e + 2 for e in n))
        b[1:-1, 1:-1, 1:-1] = g[c[0] * n[0]:(c[0] + 1) * n[0], c[1] * n[1]:(c[1] + 1) * n[1],
                                c[2] * n[2]:(c[2] + 1) * n[2]]
        blocks.append(b)
        nbr6 = []
        for a in range(3):
            for d in (-1, 1):
                cc = list(c)
                cc[a] += d
                nbr6.append(rank_of[tuple(cc)] if 0 <= cc[a] < 2 else -1)
        n26.append(nbr26_of(nbr6, lambda s, c=c: rank_of[tuple(ci + si for ci, si in zip(c, s))]))

    def box(s, recv):
        return tuple(slice(1, e + 1) if si == 0 else
                     (slice(0, 1) if recv else slice(1, 2)) if si < 0 else
                     (slice(e + 1, e + 2) if recv else slice(e, e + 1)) for si, e in zip(s, n))

    sent = {r: [(n26[r][k], blocks[r][box(dirs[k], False)].copy()) for k in range(26) if n26[r][k] >= 0]
            for r in range(8)}
    for r in range(8):
        for k in range(26):
            src = n26[r][25 - k]
            if src < 0:
                continue
            # the sender's messages to r in its send order; r's receives from src in its order
            mine = [m for dst, m in sent[src] if dst == r]
            order = [kk for kk in range(26) if n26[r][25 - kk] == src]
            blocks[r][box(dirs[25 - k], True)] = mine[order.index(k)]
    for r, c in enumerate(coords):
        want = gp[c[0] * n[0]:c[0] * n[0] + n[0] + 2, c[1] * n[1]:c[1] * n[1] + n[1] + 2,
                  c[2] * n[2]:c[2] * n[2] + n[2] + 2]
        assert np.array_equal(blocks[r], want)
    assert sum(v >= 0 for v in n26[0]) == 7


@pytest.mark.parametrize("axes,layout,ndir", [
    ([("mx", 2), ("my", 2), ("mz", 2)], {"x": "mx", "y": "my", "z": "mz"}, 7),   # cfg4
    ([("b", 2), ("mx", 2), ("my", 2)], {"batch": "b", "x": "mx", "y": "my"}, 3),  # cfg5
    ([("mx", 4)], {"x": "mx"}, 1),                                                # cfg3 (ends)
])
def test_step_nbr26_stays_inside_the_batch_coordinate(axes, layout, ndir):
    """UNetStep._nbr26 (the one-phase halo's neighbour table) on the cfg4 / cfg5 / cfg3 meshes:
    every neighbour is the rank at coordinate + s along the split spatial axes only (same
    batch coordinate), the table is symmetric (rank r at direction k of q  <=>  q at 25 - k of
    r), and a corner rank of the mesh has ``ndir`` directions."""
    from paper_1909_03108_b200.halo import directions26
    from paper_1909_03108_b200.sharding import Layout
    from paper_1909_03108_b200.step import UNetStep

    lay = Layout(layout)
    with vm.create_mesh(axes, backend="threads") as mesh:
        tables = {}
        for r in range(mesh.worker_count):
            ctx = mesh.context(r)
            nbr6 = []
            for d in ("x", "y", "z"):
                a = lay.axis_for(d)
                for s in (-1, 1):
                    n = ctx.neighbor(a, s) if a else None
                    nbr6.append(-1 if n is None else n)
            tables[r] = UNetStep._nbr26(ctx, lay, nbr6)
        dirs = directions26()
        for r, t in tables.items():
            for k, q in enumerate(t):
                if q < 0:
                    continue
                assert tables[q][25 - k] == r
                cr, cq = mesh.coords[r], mesh.coords[q]
                if "b" in mesh.axis_index:
                    assert cr[mesh.axis_index["b"]] == cq[mesh.axis_index["b"]]
                moved = {mesh.axis_index[lay.axis_for(d)]: s for d, s in zip(("x", "y", "z"), dirs[k]) if s}
                assert all(cq[i] - cr[i] == moved.get(i, 0) for i in range(len(cr)))
        assert sum(v >= 0 for v in tables[0]) == ndir
