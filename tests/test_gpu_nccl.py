"""The NCCL halo / all-reduce C ABI (csrc/halo.cu) on one GPU: a 1-rank NCCL communicator
whose rank is its own lo and hi neighbour (periodic halos — the single-GPU emulation of a
split: the same pack / NCCL group / unpack launches, no NVLink wire time).

* vm_halo_slab_fwd on a slab == numpy wrap padding of the split dims (the 3-phase protocol of
  halo.py:109-155 with every neighbour = self), bitwise, bf16 and f32; the bytes it reports
  == the analytic face bytes; vm_halo_slab_zero clears exactly the neighbour-side margins;
* the U-Net step over NCCL: the interior/boundary plane split (halo overlapped with the
  interior planes' conv on a comm stream) is bitwise the unsplit step; bucketed weight-
  gradient all-reduce on a second communicator; the whole step, NCCL calls included, captured
  in a CUDA graph and replayed bitwise the eager step.
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
from paper_1909_03108_b200.halo import nccl_comm_ptr
from paper_1909_03108_b200.step import Slab, UNetStep

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comms():
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    c1 = nccl_comm_ptr()
    g2 = dist.new_group(backend="nccl")
    c2 = nccl_comm_ptr(g2)
    yield c1, c2
    dist.destroy_process_group()


def _slab(x, dtype):
    B, D, H, W, C = x.shape
    s = Slab(B, C, D, H, W, dtype, "cuda")
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    _lib.call("vm_dense_to_slab", _lib.ptr(t), _lib.VM_F32, s.p(), _lib.dtype_code(dtype), s.bstride, B, C, D, H,
              W, 1, _lib.stream_ptr())
    return s


def _padded(s):
    """[B, D+2, H+2, W+2, CG*8] float64 copy of the whole padded slab."""
    v = s.storage[s.offset: s.offset + s.B * s.bstride].view(s.B, s.CG, s.D + 2, s.H + 2, s.W + 2, 8)
    return v.permute(0, 2, 3, 4, 1, 5).reshape(s.B, s.D + 2, s.H + 2, s.W + 2, s.CG * 8).double().cpu().numpy()


@pytest.fixture
def zero_copy_min():
    """Set the depth phase's zero-copy threshold for one test (0: always zero copy)."""
    lib = _lib.load()
    saved = []

    def set_(v):
        saved.append(lib.vm_set_halo_zero_copy_min(v))

    yield set_
    for v in saved[:1]:
        lib.vm_set_halo_zero_copy_min(v)


@pytest.mark.parametrize("zero_copy", [False, True])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("dims", [(0,), (0, 1, 2), (1, 2)])
def test_periodic_slab_halo_equals_wrap_padding(comms, zero_copy_min, dtype, dims, zero_copy):
    comm, _ = comms
    zero_copy_min(0 if zero_copy else 1 << 40)
    B, D, H, W, C = 2, 5, 6, 7, 20
    x = O.bf16_round(np.random.default_rng(3).standard_normal((B, D, H, W, C)).astype(np.float32))
    s = _slab(x, dtype)
    nbr = [-1] * 6
    for a in dims:
        nbr[2 * a] = nbr[2 * a + 1] = 0
    ws_bytes = _lib.call_size("vm_halo_slab_ws_bytes", _lib.dtype_code(dtype), B, C, D, H, W)
    ws = torch.empty(ws_bytes // 4 + 64, device="cuda")
    sent = ctypes.c_longlong(0)
    _lib.call("vm_halo_slab_fwd", ctypes.c_void_p(comm), _lib.dtype_code(dtype), s.p(), s.bstride, B, C, D, H, W,
              (ctypes.c_int * 6)(*nbr), _lib.ptr(ws), ws.numel() * 4, ctypes.byref(sent), _lib.stream_ptr())
    torch.cuda.synchronize()
    xp = np.zeros((B, D, H, W, s.CG * 8))
    xp[..., :C] = x
    # periodic along the exchanged dims, in the protocol's phase order (D, H, W)
    cur = xp
    for a in range(3):
        pad = [(0, 0)] * 5
        pad[1 + a] = (1, 1)
        cur = np.pad(cur, pad, mode="wrap" if a in dims else "constant")
    want = cur
    assert np.array_equal(_padded(s), want)
    faces = sum(2 * _lib.load().vm_halo_slab_face_bytes(_lib.dtype_code(dtype), B, C, D, H, W, a) for a in dims)
    if zero_copy and 0 in dims:  # the depth layers travel whole (padded H x W)
        faces += 2 * B * s.CG * ((H + 2) * (W + 2) - H * W) * 8 * s.storage.element_size()
    assert sent.value == faces
    _lib.call("vm_halo_slab_zero", _lib.dtype_code(dtype), s.p(), s.bstride, B, C, D, H, W, (ctypes.c_int * 6)(*nbr),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    keep = want.copy()
    for a in dims:  # neighbour sides are cleared, the rest of the shell keeps its (zero) data
        idx = [slice(None)] * 5
        for pos in (0, -1):
            idx[1 + a] = pos
            keep[tuple(idx)] = 0
    assert np.array_equal(_padded(s), keep)


def test_allreduce_single_rank_identity(comms):
    comm, _ = comms
    t = torch.arange(1000, dtype=torch.float32, device="cuda")
    _lib.call("vm_allreduce_f32", ctypes.c_void_p(comm), _lib.ptr(t), t.numel(), _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(t.cpu(), torch.arange(1000, dtype=torch.float32))


def _emulated_step(comms, params, graph, overlap):
    c1, c2 = comms
    st = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
    st.use_nccl(c1, nbr6=[0, 0, -1, -1, -1, -1], ar_comm=c2)  # depth split, periodic
    st.overlap_halo = overlap
    st.bucket_bytes = 64 << 10  # several buckets even for this small net
    return st


def test_nccl_step_overlap_buckets_and_graph_are_bitwise(comms, zero_copy_min):
    E = 32
    cfg = vm.UNetConfig(E, (16, 32), convs_per_block=2)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 6)
    img, lab = O.record_for(E, 4)
    host = (torch.from_numpy(img[None, ..., None].copy()), torch.from_numpy(lab[None].copy()))
    runs = {}
    lib = _lib.load()
    for name, overlap, zc in (("split", True, 1 << 40), ("plain", False, 1 << 40), ("zero-copy", True, 0)):
        zero_copy_min(zc)
        st = _emulated_step(comms, params, graph, overlap)
        st.overlap_min_planes = 8
        assert st.has_halo and st._split_planes(32) == overlap
        st.keep_probs = True
        st.upload(*host)
        st.forward()
        st.backward()
        torch.cuda.synchronize()
        assert len(st._grad_buckets()) > 1 and st._grads_reduced
        runs[name] = (st.probs.cpu(), st.stats.cpu(), st.grads.cpu())
    for other in ("plain", "zero-copy"):
        for a, b in zip(runs["split"], runs[other]):
            assert torch.equal(a, b), other
    # the whole step (halos, stats all-reduce, gradient buckets, SGD) in one CUDA graph
    eager = _emulated_step(comms, params, graph, True)
    capt = _emulated_step(comms, params, graph, True)
    for st in (eager, capt):
        st.overlap_min_planes = 8
        st.upload(*host)
    g = capt.capture()
    assert g is not None
    for _ in range(2):
        eager.step()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(eager.params, capt.params) and torch.equal(eager.stats, capt.stats)
    mesh.shutdown()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("dims", [(0,), (0, 1, 2), (1, 2), (0, 2)])
def test_one_phase_slab_halo_equals_wrap_padding(comms, dtype, dims):
    """vm_halo_slab_fwd26 (faces, edges and corners straight from the diagonal neighbours, one
    NCCL group) == the 3-phase protocol's slab == wrap padding, bitwise; bytes = the boxes sent."""
    from paper_1909_03108_b200.halo import directions26, nbr26_of

    comm, _ = comms
    B, D, H, W, C = 2, 5, 6, 7, 20
    x = O.bf16_round(np.random.default_rng(4).standard_normal((B, D, H, W, C)).astype(np.float32))
    nbr = [-1] * 6
    for a in dims:
        nbr[2 * a] = nbr[2 * a + 1] = 0
    n26 = nbr26_of(nbr)
    out = {}
    for name in ("one", "three"):
        s = _slab(x, dtype)
        if name == "one":
            ws_bytes = _lib.call_size("vm_halo_slab_ws_bytes26", _lib.dtype_code(dtype), B, C, D, H, W)
            ws = torch.empty(ws_bytes // 4 + 64, device="cuda")
            sent = ctypes.c_longlong(0)
            _lib.call("vm_halo_slab_fwd26", ctypes.c_void_p(comm), _lib.dtype_code(dtype), s.p(), s.bstride, B, C, D,
                      H, W, (ctypes.c_int * 26)(*n26), _lib.ptr(ws), ws.numel() * 4, ctypes.byref(sent),
                      _lib.stream_ptr())
            torch.cuda.synchronize()
            vox = sum(np.prod([e if si == 0 else 1 for si, e in zip(sd, (D, H, W))])
                      for sd, r in zip(directions26(), n26) if r >= 0)
            assert sent.value == B * s.CG * vox * 8 * s.storage.element_size()
        else:
            ws_bytes = _lib.call_size("vm_halo_slab_ws_bytes", _lib.dtype_code(dtype), B, C, D, H, W)
            ws = torch.empty(ws_bytes // 4 + 64, device="cuda")
            _lib.call("vm_halo_slab_fwd", ctypes.c_void_p(comm), _lib.dtype_code(dtype), s.p(), s.bstride, B, C, D,
                      H, W, (ctypes.c_int * 6)(*nbr), _lib.ptr(ws), ws.numel() * 4, None, _lib.stream_ptr())
            torch.cuda.synchronize()
        out[name] = _padded(s)
    xp = np.zeros((B, D, H, W, out["one"].shape[-1]))
    xp[..., :C] = x
    for a in range(3):
        pad = [(0, 0)] * 5
        pad[1 + a] = (1, 1)
        xp = np.pad(xp, pad, mode="wrap" if a in dims else "constant")
    assert np.array_equal(out["one"], xp)
    assert np.array_equal(out["one"], out["three"])


def test_nccl_step_3d_mesh_one_phase_is_bitwise_three_phase(comms, monkeypatch):
    """The U-Net step on a periodic 2x2x2-style emulation (every dim split, every neighbour =
    this rank): one-phase halo (vm_halo_slab_fwd26) == 3-phase halo, bitwise, eager and graph."""
    E = 32
    cfg = vm.UNetConfig(E, (16, 32), convs_per_block=2)
    mesh = vm.create_mesh([("one", 1)])
    graph = vm.build(cfg, mesh, {})
    params = vm.init_params(graph, 6)
    img, lab = O.record_for(E, 4)
    host = (torch.from_numpy(img[None, ..., None].copy()), torch.from_numpy(lab[None].copy()))
    c1, c2 = comms
    runs = {}
    for phases in ("1", "3"):
        monkeypatch.setenv("VOXMESH_HALO_PHASES", phases)
        st = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
        st.use_nccl(c1, nbr6=[0] * 6, ar_comm=c2)
        assert (st.halo.nbr26 is not None) == (phases == "1")
        st.keep_probs = True
        st.upload(*host)
        g = st.capture()
        assert g is not None
        g.replay()
        torch.cuda.synchronize()
        runs[phases] = (st.probs.cpu(), st.stats.cpu(), st.grads.cpu(), st.params.cpu())
    for a, b in zip(runs["1"], runs["3"]):
        assert torch.equal(a, b)
    mesh.shutdown()
