"""Host-side protocol of the peer-memory depth halo (halo.PeerDepthHalo) across ranks, on CPU:
gloo, one process per rank, world size 3 (rank 0 and 2 at the global boundary).  The CUDA-IPC
calls are replaced by a fake mapping (a peer address = its rank tag | its local address), so the
test checks what the kernels would be handed, not the copies themselves (those are the GPU
tests, with every neighbour = self):

* connect() maps each exchanged slab to the neighbours' copies of the SAME slab (program
  order), and the neighbours' flag words;
* for every exchange slot, the word a rank's producer signals on its lo neighbour is that
  neighbour's "from hi" own word, and on its hi neighbour that neighbour's "from lo" word, and
  it waits on exactly the sides it pushes to: the flag graph is symmetric, so every wait has a
  matching signal (no rank can wait forever);
* fused (reserve_push / consume) and standalone exchanges consume slots in the same program
  order on every rank."""

import os
import socket
import struct
import sys
import traceback

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = 1 << 56


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    try:
        sys.path.insert(0, ROOT)
        import ctypes

        import torch
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1909_03108_b200 import _lib, halo as H
        from paper_1909_03108_b200.step import Slab

        calls = []

        def fake_call(name, *args):
            if name == "vm_ipc_handle":  # (ptr, handle64*, offset*): handle = (rank, ptr)
                ptr = args[0].value if isinstance(args[0], ctypes.c_void_p) else int(args[0])
                ctypes.memmove(args[1], struct.pack("<qq", rank, ptr) + bytes(48), 64)
                ctypes.c_int64.from_address(args[2]).value = 0
                return 0
            if name == "vm_ipc_open":  # (handle64*, base*): a tagged address of the owner
                r, ptr = struct.unpack("<qq", ctypes.string_at(args[0], 16))
                ctypes.c_void_p.from_address(args[1]).value = (r + 1) * TAG | ptr
                return 0
            calls.append((name, args))
            return 0

        _lib.call = fake_call
        H._lib.call = fake_call
        H._lib.stream_ptr = lambda stream=None: None  # no CUDA stream on the CPU box
        nbr6 = [rank - 1 if rank > 0 else -1, rank + 1 if rank < world - 1 else -1, -1, -1, -1, -1]
        slabs = [Slab(1, c, 4, 5, 6, torch.float32, "cpu") for c in (8, 16, 24)]
        halo = H.PeerDepthHalo(nbr6, "cpu", self_peers=False)
        halo.connect(slabs)
        own = halo.state.data_ptr()
        mine = [s.ptr for s in slabs]
        everyone = [None] * world
        dist.all_gather_object(everyone, {"state": own, "slabs": mine})
        res = {"ok": True, "msgs": []}

        def check(cond, msg):
            if not cond:
                res["ok"] = False
                res["msgs"].append(msg)

        for side, r in (("lo", nbr6[0]), ("hi", nbr6[1])):
            i = 0 if side == "lo" else 1
            if r < 0:
                check(halo.peer_state[i] is None, f"{side}: state mapped at a boundary")
                continue
            check(halo.peer_state[i] == (r + 1) * TAG | everyone[r]["state"], f"{side}: neighbour state")
            for k, s in enumerate(slabs):
                check(halo.peer_slab[s.ptr][i] == (r + 1) * TAG | everyone[r]["slabs"][k], f"{side}: slab {k}")
        # a step: fused push of slab 0, standalone exchange of slab 1, fused push of slab 2
        halo.begin_step()
        plan = []
        p0 = halo.reserve_push(slabs[0])
        w0 = halo.consume(slabs[0])
        halo.consume(slabs[1])  # standalone -> vm_halo_depth_push
        p2 = halo.reserve_push(slabs[2])
        w2 = halo.consume(slabs[2])
        push_calls = [a for n, a in calls if n == "vm_halo_depth_push"]
        check(len(push_calls) == 1, "one standalone push")
        for slot, p, w in ((0, p0, w0), (2, p2, w2)):
            # own words of this slot: [from lo, from hi]
            check(w["wait_own"] == own + 4 * (8 + 2 * slot), f"slot {slot}: own words")
            check(w["wait_lo"] == int(nbr6[0] >= 0) and w["wait_hi"] == int(nbr6[1] >= 0), "waits on pushed sides")
            if nbr6[0] >= 0:  # signal the lo neighbour's "from hi" word
                lo = nbr6[0]
                check(p["lo_flag"] == (lo + 1) * TAG | (everyone[lo]["state"] + 4 * (8 + 2 * slot + 1)),
                      f"slot {slot}: lo flag")
            else:
                check(p["lo_flag"] is None and p["push_lo"] is None, "no lo push at the boundary")
            if nbr6[1] >= 0:
                hi = nbr6[1]
                check(p["hi_flag"] == (hi + 1) * TAG | (everyone[hi]["state"] + 4 * (8 + 2 * slot)),
                      f"slot {slot}: hi flag")
            else:
                check(p["hi_flag"] is None and p["push_hi"] is None, "no hi push at the boundary")
        plan.append(halo._slot)
        out[rank] = res
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out[rank] = {"ok": False, "msgs": [traceback.format_exc()]}


def test_peer_halo_protocol_world3():
    world = 3
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        assert res[r]["ok"], (r, res[r]["msgs"])
