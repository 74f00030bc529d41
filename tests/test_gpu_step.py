"""GPU parity of the slab train-step program against the f64 oracle."""

import numpy as np
import pytest
import torch

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200.step import UNetStep
from tests.helpers import oracle_step, rel_l2

pytestmark = pytest.mark.gpu


def _setup(extent=16, filters=(8, 16), cpb=2, seed=1):
    cfg = vm.UNetConfig(extent, filters, convs_per_block=cpb)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, seed)
    img, labels = O.record_for(extent, 0)
    x = img[None, ..., None]
    oh = O.one_hot(labels[None], 3)
    return mesh, graph, params, x, oh


def _run(graph, params, x, oh, dtype, impl):
    st = UNetStep(graph, params, dtype=dtype, conv_impl=impl, device="cuda")
    st.keep_probs = True
    st.load_inputs(torch.from_numpy(x).cuda(), torch.from_numpy(oh).cuda())
    st.forward()
    st.backward()
    torch.cuda.synchronize()
    probs = st.probs.reshape(oh.shape).cpu().numpy()
    return st, probs, st.stats.cpu().numpy(), st.grad_dict()


@pytest.mark.parametrize("impl", ["simt"])
def test_fp32_step_matches_f64_oracle(impl):
    mesh, graph, params, x, oh = _setup()
    st, probs, stats, grads = _run(graph, params, x, oh, torch.float32, impl)
    rprobs, rstats, rgrads, _ = oracle_step(graph, params, x, oh)
    assert rel_l2(probs, rprobs) <= 1e-5
    assert rel_l2(stats, rstats) <= 1e-5
    worst = max(max(rel_l2(grads[k][0], rgrads[k][0]), rel_l2(grads[k][1], rgrads[k][1])) for k in rgrads)
    assert worst <= 1e-5, worst
    mesh.shutdown()


def test_bf16_step_close_to_oracle():
    mesh, graph, params, x, oh = _setup()
    st, probs, stats, grads = _run(graph, params, x, oh, torch.bfloat16, "simt")
    rprobs, rstats, rgrads, _ = oracle_step(graph, params, x, oh)
    assert rel_l2(probs, rprobs) <= 1e-2
    assert rel_l2(stats, rstats) <= 1e-2
    mesh.shutdown()


def test_tc_step_matches_simt_step_and_oracle():
    mesh, graph, params, x, oh = _setup(extent=16, filters=(16, 32), cpb=2)
    st, probs, stats, grads = _run(graph, params, x, oh, torch.bfloat16, "tc")
    _, probs_s, stats_s, grads_s = _run(graph, params, x, oh, torch.bfloat16, "simt")
    rprobs, rstats, rgrads, _ = oracle_step(graph, params, x, oh)
    assert rel_l2(probs, rprobs) <= 1e-2
    assert rel_l2(stats, rstats) <= 1e-2
    assert rel_l2(probs, probs_s) <= 1e-2
    # end-to-end bf16 weight grads are storage-bound (~2-5e-2 vs f64)
    worst = max(rel_l2(grads[k][0], rgrads[k][0]) for k in rgrads)
    assert worst <= 1e-1, worst
    mesh.shutdown()
