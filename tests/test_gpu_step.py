"""GPU parity of the slab train-step program against the f64 oracle."""

import numpy as np
import pytest
import torch

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200.step import UNetStep
from tests.helpers import node_tuples, oracle_step, rel_l2

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


def test_tc_step_32cube_exercises_thin_kernels():
    # W >= 32 and Cout <= 32: the kd-stacked sweep fwd/dgrad and the kd-along-N wgrad run
    mesh, graph, params, x, oh = _setup(extent=32, filters=(16, 32), cpb=2, seed=3)
    st, probs, stats, grads = _run(graph, params, x, oh, torch.bfloat16, "tc")
    rprobs, rstats, rgrads, _ = oracle_step(graph, params, x, oh)
    assert rel_l2(probs, rprobs) <= 1e-2
    assert rel_l2(stats, rstats) <= 1e-2
    worst = max(rel_l2(grads[k][0], rgrads[k][0]) for k in rgrads)
    assert worst <= 1e-1, worst
    worst_b = max(rel_l2(grads[k][1], rgrads[k][1]) for k in rgrads)
    assert worst_b <= 1e-1, worst_b
    mesh.shutdown()


def test_tc_step_wide_ladder():
    # cfg3/cfg4-style ladder (to 256 channels): chunked wide wgrad, multi-chunk fwd/dgrad
    mesh, graph, params, x, oh = _setup(extent=16, filters=(32, 64, 128, 256), cpb=1, seed=5)
    st, probs, stats, grads = _run(graph, params, x, oh, torch.bfloat16, "tc")
    rprobs, rstats, rgrads, _ = oracle_step(graph, params, x, oh)
    assert rel_l2(probs, rprobs) <= 1e-2
    assert rel_l2(stats, rstats) <= 1e-2
    worst = max(rel_l2(grads[k][0], rgrads[k][0]) for k in rgrads)
    assert worst <= 1e-1, worst
    mesh.shutdown()


def test_train_step_host_prefetch_is_bitwise_the_plain_path():
    # the copy-stream prefetch of step k+1's inputs must not change any result
    extent = 32
    cfg = vm.UNetConfig(extent, (16, 32), convs_per_block=2)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 5)
    recs = [O.record_for(extent, i) for i in range(2)]
    host = [(torch.from_numpy(img[None, ..., None].copy()).pin_memory(),
             torch.from_numpy(lab[None].copy()).pin_memory()) for img, lab in recs]
    a = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
    b = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
    la, lb = [], []
    for k in range(4):
        cur, nxt = host[k % 2], host[(k + 1) % 2]
        la.append(a.train_step_host(cur[0], cur[1], next_inputs=nxt if k < 3 else None))
        b.upload(cur[0], cur[1])
        b.step()
        lb.append(b.loss()[0])
    torch.cuda.synchronize()
    assert la == lb
    pa, pb = a.param_dict(), b.param_dict()
    for k in pa:
        assert np.array_equal(pa[k]["kernel"], pb[k]["kernel"]) and np.array_equal(pa[k]["bias"], pb[k]["bias"])
    mesh.shutdown()


def test_train_loop_host_matches_step_by_step():
    extent = 32
    cfg = vm.UNetConfig(extent, (16, 32), convs_per_block=2)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 9)
    recs = [O.record_for(extent, i) for i in range(3)]
    host = [(torch.from_numpy(img[None, ..., None].copy()).pin_memory(),
             torch.from_numpy(lab[None].copy()).pin_memory()) for img, lab in recs]
    a = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
    b = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
    la = a.train_loop_host(host)
    lb = [b.train_step_host(*h) for h in host]
    assert [x[0] for x in la] == lb
    pa, pb = a.param_dict(), b.param_dict()
    for k in pa:
        assert np.array_equal(pa[k]["kernel"], pb[k]["kernel"])
    mesh.shutdown()


@pytest.mark.parametrize("filters", [(64, 128), (128, 256)])
def test_tc_step_wide_base_head(filters):
    # 64/128-channel head input: the fixed head fwd/bwd kernels for wide first levels
    mesh, graph, params, x, oh = _setup(extent=16, filters=filters, cpb=1, seed=7)
    st, probs, stats, grads = _run(graph, params, x, oh, torch.bfloat16, "tc")
    rprobs, rstats, rgrads, _ = oracle_step(graph, params, x, oh)
    assert rel_l2(probs, rprobs) <= 1e-2
    assert rel_l2(stats, rstats) <= 1e-2
    head = [k for k in rgrads if k.startswith("head")]
    for k in head:
        assert rel_l2(grads[k][0], rgrads[k][0]) <= 2e-2, k
        assert rel_l2(grads[k][1], rgrads[k][1]) <= 2e-2, k
    worst = max(rel_l2(grads[k][0], rgrads[k][0]) for k in rgrads)
    assert worst <= 1e-1, worst
    mesh.shutdown()


@pytest.mark.parametrize("ncls,dice", [(2, (1,)), (4, (1, 2))])
def test_tc_step_other_class_counts(ncls, dice):
    # 2 and 4 classes: the fixed head kernels' other instantiations against the oracle
    cfg = vm.UNetConfig(16, (16, 32), convs_per_block=1, num_classes=ncls)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 2)
    img, labels = O.record_for(16, 0)
    labels = np.minimum(labels, ncls - 1).astype(labels.dtype)
    x = img[None, ..., None]
    oh = O.one_hot(labels[None], ncls)
    st = UNetStep(graph, params, dtype=torch.bfloat16, conv_impl="tc", device="cuda", dice_classes=dice)
    st.keep_probs = True
    st.load_inputs(torch.from_numpy(x).cuda(), torch.from_numpy(oh).cuda())
    st.forward()
    st.backward()
    torch.cuda.synchronize()
    probs = st.probs.reshape(oh.shape).cpu().numpy()
    stats, grads = st.stats.cpu().numpy(), st.grad_dict()
    p64 = {k: {"kernel": np.asarray(v["kernel"], np.float64), "bias": np.asarray(v["bias"], np.float64)}
           for k, v in params.items()}
    rprobs, tape, _ = O.oracle_forward(node_tuples(graph), p64, x.astype(np.float64))
    rstats = O.loss_stats(rprobs, oh.astype(np.float64))
    dprobs = O.loss_grad(rprobs, oh.astype(np.float64), rstats, int(np.prod(x.shape[:4])), dice_classes=dice)
    rgrads, _ = O.oracle_backward(node_tuples(graph), p64, tape, dprobs)
    assert rel_l2(probs, rprobs) <= 1e-2
    assert rel_l2(stats, rstats) <= 1e-2
    worst = max(rel_l2(grads[k][0], rgrads[k][0]) for k in rgrads)
    assert worst <= 1e-1, worst
    mesh.shutdown()


@pytest.mark.parametrize("C,ncls,dprobs", [(16, 3, False), (32, 3, False), (16, 2, False), (32, 4, False),
                                           (16, 3, True), (32, 3, True)])
def test_head_bwd_team_kernel_matches_group_kernel(C, ncls, dprobs):
    # rows of 32+ voxels take the team kernel (softmax once per voxel, reduce-scattered logits);
    # the per-group kernel is the reference: same gradients and head-weight partial sums
    from paper_1909_03108_b200 import _lib
    from paper_1909_03108_b200.step import Slab

    lib = _lib.load()
    torch.manual_seed(C + ncls)
    B, D, H, W = 2, 3, 5, 64
    y = Slab(B, C, D, H, W, torch.bfloat16, "cuda")
    y.storage.normal_()
    w = torch.randn(C * ncls, device="cuda") * 0.3
    b = torch.randn(ncls, device="cuda") * 0.1
    nvox = B * D * H * W
    lab = torch.randint(0, ncls, (nvox,), dtype=torch.uint8, device="cuda")
    stats = torch.rand(3 * ncls + 1, device="cuda") * 100 + 1
    dp = torch.randn(nvox * ncls, device="cuda")
    nb = int(lib.vm_head_partials_count(B, D, H, W))
    out = {}
    for team in (0, 1):
        lib.vm_debug_set_head_team(team)
        g = Slab(B, C, D, H, W, torch.bfloat16, "cuda")
        wp = torch.zeros(nb * (C * ncls + ncls), device="cuda")
        if dprobs:
            _lib.call("vm_head_bwd_dprobs", _lib.VM_BF16, y.p(), y.bstride, _lib.ptr(w), _lib.ptr(b), _lib.ptr(dp),
                      g.p(), g.bstride, _lib.ptr(wp), B, C, ncls, D, H, W, 1, _lib.stream_ptr())
        else:
            _lib.call("vm_head_bwd", _lib.VM_BF16, y.p(), y.bstride, _lib.ptr(w), _lib.ptr(b), _lib.ptr(lab),
                      _lib.ptr(stats), g.p(), g.bstride, _lib.ptr(wp), B, C, ncls, D, H, W, 0.9, 0.1, float(nvox),
                      (1 << ncls) - 2, 1e-12, 1, _lib.stream_ptr())
        torch.cuda.synchronize()
        out[team] = (g.interior().float().cpu().numpy(), wp.view(nb, -1).double().sum(0).cpu().numpy())
    lib.vm_debug_set_head_team(1)
    # bf16 outputs: the logits are summed in another order, so a few elements round the other way
    assert rel_l2(out[1][0], out[0][0]) <= 1e-3
    assert rel_l2(out[1][1], out[0][1]) <= 1e-5
    assert np.abs(out[1][0]).max() > 0


@pytest.mark.parametrize("C,ncls", [(32, 3), (32, 2), (32, 4)])
def test_head_fwd_team_kernel_matches_voxel_kernel(C, ncls):
    # 32-channel rows of 32+ voxels take the team forward kernel: probabilities, argmax, loss-statistic
    # partial sums and the label-range flag as the one-thread-per-voxel kernel gives them
    from paper_1909_03108_b200 import _lib
    from paper_1909_03108_b200.step import Slab

    lib = _lib.load()
    torch.manual_seed(C * ncls)
    B, D, H, W = 2, 3, 4, 96
    y = Slab(B, C, D, H, W, torch.bfloat16, "cuda")
    y.storage.normal_()
    w = torch.randn(C * ncls, device="cuda") * 0.3
    b = torch.randn(ncls, device="cuda") * 0.1
    nvox = B * D * H * W
    nb = int(lib.vm_head_partials_count(B, D, H, W))
    for bad in (False, True):
        lab = torch.randint(0, ncls, (nvox,), dtype=torch.uint8, device="cuda")
        if bad:
            lab[nvox // 3] = ncls
        out = {}
        for team in (0, 1):
            lib.vm_debug_set_head_team(team)
            err = torch.zeros(1, dtype=torch.int32, device="cuda")
            probs = torch.zeros(nvox * ncls, device="cuda")
            pred = torch.zeros(nvox, dtype=torch.uint8, device="cuda")
            part = torch.zeros(nb * (3 * ncls + 1), device="cuda")
            _lib.call("vm_head_fwd", _lib.VM_BF16, y.p(), y.bstride, _lib.ptr(w), _lib.ptr(b), _lib.ptr(lab),
                      _lib.ptr(err), _lib.ptr(probs), _lib.ptr(pred), _lib.ptr(part), B, C, ncls, D, H, W, 1e-12,
                      _lib.stream_ptr())
            torch.cuda.synchronize()
            out[team] = (probs.cpu().numpy(), pred.cpu().numpy(), part.view(nb, -1).double().sum(0).cpu().numpy(),
                         int(err.item()))
        lib.vm_debug_set_head_team(1)
        assert rel_l2(out[1][0], out[0][0]) <= 1e-6
        assert (out[1][1] != out[0][1]).mean() <= 1e-3  # argmax ties may resolve differently at ulp level
        assert rel_l2(out[1][2], out[0][2]) <= 1e-5
        assert out[1][3] == out[0][3] == int(bad)
