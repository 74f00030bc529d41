"""A/B of the emulated depth-split halo (bench.py's N=1 emulation) on one GPU: step time of a
cfg3 K-way rank block with the exchange off, on without the plane split, and on with the split
at several minimum plane counts; plus the per-exchange cost of the C-ABI halo alone."""
import os, socket, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import paper_1909_03108_b200 as vm
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.data import synth_record
from paper_1909_03108_b200.halo import nccl_comm_ptr
from paper_1909_03108_b200.step import UNetStep

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=torch.device("cuda", 0))
comm = nccl_comm_ptr(); ar = nccl_comm_ptr(dist.new_group(backend="nccl"))
E = 256
cfg = vm.recipe_for_resolution(E, 0.5)
mesh = vm.create_mesh([("one", 1)], backend="threads")
graph = vm.build(cfg, mesh, {})
params = vm.init_params(graph, 1)
loc = (E // K, E, E)
st = UNetStep(graph, params, dtype=torch.bfloat16, global_shape=(E, E, E), local_shape=loc)
st.use_nccl(comm, nbr6=[0, 0, -1, -1, -1, -1], ar_comm=ar)
img, lab = synth_record(E, 7, 0)
st.upload(torch.from_numpy(img[None, :loc[0], ..., None].copy()), torch.from_numpy(lab[None, :loc[0]].copy()))
for _ in range(2): st.step()
torch.cuda.synchronize()

def timeit(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n

def variant(halo, overlap, minp=8, reserve=8, eager=False):
    st.has_halo = halo; st.overlap_halo = overlap; st.overlap_min_planes = minp; st.halo_sm_reserve = reserve
    if eager:
        return timeit(st.step)
    g = st.capture()
    t = timeit(g.replay)
    del g
    return t

print(f"eager: no halo {variant(False, False, eager=True):.3f}  halo no split {variant(True, False, eager=True):.3f}  "
      f"split D>=16 r8 {variant(True, True, 16, 8, eager=True):.3f} ms")

print(f"K={K} block {loc}")
print(f"no halo                 {variant(False, False):.3f} ms")
print(f"halo, no split          {variant(True, False):.3f} ms")
for m in (16, 32):
    for r in (4, 8, 16):
        print(f"halo, split D>={m:<3d} reserve {r:2d} SMs   {variant(True, True, m, r):.3f} ms")
# the exchange alone per conv input slab
st.has_halo = True
rows = []
for n in graph.nodes:
    if n.op == "conv" and n.k == 3:
        x = st.out[n.inputs[0]]
        t = timeit(lambda: st.halo.forward(x), 20)
        rows.append((n.id, x.D, x.C, t * 1e3))
tot = sum(r[3] for r in rows)
_lib.load().vm_debug_halo_loopback(1)
lb = 0.0
for n in graph.nodes:
    if n.op == "conv" and n.k == 3:
        x = st.out[n.inputs[0]]
        lb += timeit(lambda: st.halo.forward(x), 20) * 1e3
print(f"exchange alone with device-copy loopback instead of NCCL: {lb:.0f} us")
print(f"step with loopback transport: no split {variant(True, False):.3f} ms, split D>=16 r8 {variant(True, True, 16, 8):.3f} ms")
_lib.load().vm_debug_halo_loopback(0)
print(f"exchange alone, sum over forward conv inputs: {tot:.0f} us ({len(rows)} exchanges)")
for r in rows[:6] + rows[-4:]:
    print("  %-12s D=%-3d C=%-4d %.1f us" % r)
dist.destroy_process_group()
