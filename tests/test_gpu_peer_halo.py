"""The peer-memory depth halo (vm_halo_depth_push, halo.PeerDepthHalo) on one GPU, with every
neighbour = this rank (the periodic single-GPU emulation of a depth split):

* one push == numpy wrap padding of the depth dim, bitwise, bf16 and f32, several samples;
  the H / W margins stay zero; repeated exchanges under a bumped epoch stay correct;
* the weight-gradient kernels never read a depth margin layer of gy: garbage in gy's margin
  layers leaves gw / gb bitwise unchanged (kd and general kernels) — the property that lets
  wgrad run concurrently with the exchange that fills them;
* the U-Net step over the peer transport (wgrad concurrent with exchange + dgrad) is bitwise
  the step over NCCL (pack / NCCL / unpack, serial), eager and captured in a CUDA graph.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch

import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.halo import PeerDepthHalo, nccl_comm_ptr
from paper_1909_03108_b200.step import Slab, UNetStep

pytestmark = pytest.mark.gpu


def _slab(x, dtype):
    B, D, H, W, C = x.shape
    s = Slab(B, C, D, H, W, dtype, "cuda")
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    _lib.call("vm_dense_to_slab", _lib.ptr(t), _lib.VM_F32, s.p(), _lib.dtype_code(dtype), s.bstride, B, C, D, H,
              W, 1, _lib.stream_ptr())
    return s


def _padded(s):
    v = s.storage[s.offset: s.offset + s.B * s.bstride].view(s.B, s.CG, s.D + 2, s.H + 2, s.W + 2, 8)
    return v.permute(0, 2, 3, 4, 1, 5).reshape(s.B, s.D + 2, s.H + 2, s.W + 2, s.CG * 8).double().cpu().numpy()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_depth_push_equals_wrap_padding(dtype):
    sides = (0, 0)  # a rank that is its own lo neighbour is its own hi neighbour too
    B, D, H, W, C = 2, 5, 6, 7, 20
    rng = np.random.default_rng(11)
    halo = PeerDepthHalo([sides[0], sides[1], -1, -1, -1, -1], "cuda")
    for rep in range(3):  # a fresh epoch each time: the flags of the previous round must not satisfy the wait
        x = O.bf16_round(rng.standard_normal((B, D, H, W, C)).astype(np.float32))
        s = _slab(x, dtype)
        halo.begin_step()
        halo.forward(s)
        torch.cuda.synchronize()
        xp = np.zeros((B, D, H, W, s.CG * 8))
        xp[..., :C] = x
        want = np.pad(xp, [(0, 0), (1, 1), (1, 1), (1, 1), (0, 0)])
        if sides[1] >= 0:  # our hi neighbour (self) pushed its layer D into its layer 0... and ours
            want[:, 0] = want[:, D]
        if sides[0] >= 0:
            want[:, D + 1] = want[:, 1]
        got = _padded(s)
        assert np.array_equal(got, want), rep
        epoch = int(halo.state[0].item())
        assert epoch == rep + 1
        own = halo.state[8:10].cpu().tolist()
        assert own == [epoch, epoch]
        halo.check()


@pytest.mark.parametrize("shape", [(1, 16, 16, 5, 6, 40), (1, 32, 32, 4, 4, 64), (2, 16, 48, 3, 5, 34),
                                   (1, 64, 64, 4, 6, 34), (1, 32, 256, 4, 6, 8), (1, 16, 16, 4, 4, 8)])
def test_wgrad_ignores_gy_depth_margins(shape):
    B, cin, cout, D, H, W = shape
    rng = np.random.default_rng(7 + sum(shape))
    x = O.bf16_round(rng.standard_normal((B, D, H, W, cin)).astype(np.float32))
    g = O.bf16_round(rng.standard_normal((B, D, H, W, cout)).astype(np.float32))
    xs, gs = _slab(x, torch.bfloat16), _slab(g, torch.bfloat16)

    def wgrad():
        gw = torch.zeros(27 * cin * cout, device="cuda")
        gb = torch.zeros(cout, device="cuda")
        nb = _lib.call_size("vm_conv3d_wgrad_tc_ws", B, cin, cout, D, H, W)
        ws = torch.empty(nb // 4 + 64, device="cuda")
        _lib.call("vm_conv3d_wgrad_tc", xs.p(), xs.bstride, gs.p(), gs.bstride, _lib.ptr(gw), _lib.ptr(gb),
                  _lib.ptr(ws), B, cin, cout, D, H, W, _lib.stream_ptr())
        torch.cuda.synchronize()
        return gw.cpu(), gb.cpu()

    ref = wgrad()
    v = gs.storage[: B * gs.bstride].view(B, gs.CG, D + 2, (H + 2) * (W + 2) * 8)
    junk = torch.from_numpy(O.bf16_round(rng.standard_normal(v[:, :, 0].shape).astype(np.float32) * 5)).cuda()
    v[:, :, 0] = junk.to(torch.bfloat16)
    v[:, :, D + 1] = junk.flip(-1).to(torch.bfloat16)
    got = wgrad()
    assert torch.equal(ref[0], got[0]) and torch.equal(ref[1], got[1])


@pytest.fixture(scope="module")
def comms():
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    c1 = nccl_comm_ptr()
    c2 = nccl_comm_ptr(dist.new_group(backend="nccl"))
    yield c1, c2
    dist.destroy_process_group()


def test_peer_step_equals_nccl_step_eager_and_graph(comms):
    E = 32
    cfg = vm.UNetConfig(E, (16, 32), convs_per_block=2)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 6)
    img, lab = O.record_for(E, 4)
    host = (torch.from_numpy(img[None, ..., None].copy()), torch.from_numpy(lab[None].copy()))
    nbr6 = [0, 0, -1, -1, -1, -1]

    def make(kind):
        st = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
        if kind == "nccl":
            st.use_nccl(comms[0], nbr6=nbr6, ar_comm=comms[1])
            st.overlap_halo = False
        else:
            st.use_peer_halo(nbr6=nbr6)
        st.keep_probs = True
        st.upload(*host)
        return st

    runs = {}
    for kind in ("nccl", "peer"):
        st = make(kind)
        assert st.has_halo
        st.forward()
        st.backward()
        st.all_reduce_grads()
        torch.cuda.synchronize()
        runs[kind] = (st.probs.cpu(), st.stats.cpu(), st.grads.cpu())
    for a, b in zip(runs["nccl"], runs["peer"]):
        assert torch.equal(a, b)
    eager, capt = make("peer"), make("peer")
    g = capt.capture()
    assert g is not None
    for _ in range(3):
        eager.step()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(eager.params, capt.params) and torch.equal(eager.stats, capt.stats)
    assert int(capt.halo.state[0].item()) >= 3


def test_fused_push_step_equals_standalone_push_step():
    # the producer convs push their boundary layers from the epilogue (vm_conv3d_fwd_tc_link)
    # == every exchange as a standalone vm_halo_depth_push; eager and graph; several levels
    E = 32
    cfg = vm.UNetConfig(E, (16, 32, 64), convs_per_block=2)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 3)
    img, lab = O.record_for(E, 2)
    host = (torch.from_numpy(img[None, ..., None].copy()), torch.from_numpy(lab[None].copy()))

    def make(fuse):
        st = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
        st.use_peer_halo(nbr6=[0, 0, -1, -1, -1, -1])
        st.fuse_halo = fuse
        st.keep_probs = True
        st.upload(*host)
        return st

    runs = {}
    for fuse in (False, True):
        st = make(fuse)
        st.forward()
        st.backward()
        torch.cuda.synchronize()
        st.halo.check()
        if fuse:
            assert len(st._links) > 0  # fused links were used
        runs[fuse] = (st.probs.cpu(), st.stats.cpu(), st.grads.cpu())
    for a, b in zip(runs[False], runs[True]):
        assert torch.equal(a, b)
    eager, capt = make(True), make(True)
    g = capt.capture()
    for _ in range(3):
        eager.step()
        g.replay()
    torch.cuda.synchronize()
    capt.halo.check()
    assert torch.equal(eager.params, capt.params) and torch.equal(eager.stats, capt.stats)


def test_ipc_connect_failure_is_collective_and_clean(comms):
    # a CUDA-IPC handle cannot be opened by the process that exported it: connect() must
    # report a HaloError on every rank (here: the only one) instead of leaving a half-mapped
    # transport, so the caller can fall back to NCCL together
    from paper_1909_03108_b200.errors import HaloError

    s = Slab(1, 16, 4, 6, 8, torch.bfloat16, "cuda")
    halo = PeerDepthHalo([0, 0, -1, -1, -1, -1], "cuda", self_peers=False)
    with pytest.raises(HaloError):
        halo.connect([s])
