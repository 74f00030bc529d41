"""Spatially partitioned train step on one GPU: the threads mesh runs one UNetStep per rank
(own CUDA stream, halo exchange through the pack/unpack kernels, gradient and loss-statistics
all-reduce), against the unpartitioned step on the same global volume.

SURVEY §8(c) property tests: mesh independence (`test_acceptance.py:171-196`) and
distributed-vs-dense conv backward (`test_ops.py:130-143`).  The forward is the same
arithmetic per voxel, so probabilities agree bitwise up to the loss normalisation; weight
gradients differ only in the order of the per-rank partial sums."""

import numpy as np
import pytest
import torch

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200.step import UNetStep
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu


def _single(cfg, params, img, lab):
    mesh = vm.create_mesh([("one", 1)])
    g = vm.build(cfg, mesh, {})
    st = UNetStep(g, params, dtype=torch.bfloat16, device="cuda")
    st.upload(torch.from_numpy(img[None, ..., None].copy()), torch.from_numpy(lab[None].copy()))
    st.forward()
    st.backward()
    torch.cuda.synchronize()
    out = st.loss()[0], st.grad_dict()
    mesh.shutdown()
    return out


@pytest.mark.parametrize("axes,layout", [
    ([("mx", 2)], {"x": "mx"}),
    ([("mx", 2), ("my", 2)], {"x": "mx", "y": "my"}),
])
def test_partitioned_step_matches_unpartitioned(axes, layout):
    E = 32
    cfg = vm.UNetConfig(E, (16, 32), convs_per_block=2)
    mesh1 = vm.create_mesh([("one", 1)])
    params = vm.init_params(vm.build(cfg, mesh1, {}), 4)
    mesh1.shutdown()
    img, lab = O.record_for(E, 1)
    loss1, grads1 = _single(cfg, params, img, lab)

    mesh = vm.create_mesh(axes, backend="threads")
    g = vm.build(cfg, mesh, layout)
    div = [mesh.axis_size(layout[d]) if d in layout else 1 for d in ("x", "y", "z")]
    loc = tuple(E // d for d in div)
    blocks_img, blocks_lab = [], []
    for coord in mesh.coords:
        c = [coord[mesh.axis_index[layout[d]]] if d in layout else 0 for d in ("x", "y", "z")]
        sl = tuple(slice(ci * n, (ci + 1) * n) for ci, n in zip(c, loc))
        blocks_img.append(torch.from_numpy(img[sl][None, ..., None].copy()))
        blocks_lab.append(torch.from_numpy(lab[sl][None].copy()))

    def work(ctx, im, lb):
        st = UNetStep(g, params, ctx=ctx, dtype=torch.bfloat16, global_shape=(E, E, E), local_shape=loc)
        st.overlap_min_planes = 8  # exercise the interior/boundary plane split (host transport)
        st.upload(im, lb)
        st.forward()
        st.backward()
        st.all_reduce_grads()
        torch.cuda.synchronize()
        return st.loss()[0], st.grad_dict(), ctx.counters["p2p_bytes"]

    res = mesh.run(work, per_worker=(blocks_img, blocks_lab))
    mesh.shutdown()
    for loss, grads, nbytes in res:
        assert abs(loss - loss1) <= 1e-5 * abs(loss1)
        assert nbytes > 0
        worst = max(max(rel_l2(grads[k][0], grads1[k][0]), rel_l2(grads[k][1], grads1[k][1])) for k in grads1)
        assert worst <= 1e-3, worst
    # every rank holds the same all-reduced gradient, bitwise
    g0 = res[0][1]
    for _, grads, _ in res[1:]:
        for k in g0:
            assert np.array_equal(grads[k][0], g0[k][0]) and np.array_equal(grads[k][1], g0[k][1])
