"""Forward of the NCCL-emulated depth split with and without the interior/boundary split:
first diverging activation slab, with PDL on and off."""
import os, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import paper_1909_03108_b200 as vm
from oracle import voxmesh_oracle as O
from paper_1909_03108_b200 import _lib
from paper_1909_03108_b200.halo import nccl_comm_ptr
from paper_1909_03108_b200.step import UNetStep

with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=torch.device("cuda", 0))
c1 = nccl_comm_ptr()
E = 32
cfg = vm.UNetConfig(E, (16, 32), convs_per_block=2)
mesh = vm.create_mesh([("one", 1)])
graph = vm.build(cfg, mesh, {})
params = vm.init_params(graph, 6)
img, lab = O.record_for(E, 4)
host = (torch.from_numpy(img[None, ..., None].copy()), torch.from_numpy(lab[None].copy()))
def run(overlap, pdl, comm_mode):
    st = UNetStep(graph, params, dtype=torch.bfloat16, device="cuda")
    if comm_mode:
        st.use_nccl(c1, nbr6=[0, 0, -1, -1, -1, -1])
    st.overlap_halo = overlap
    st.pdl_forward = pdl
    st.keep_probs = True
    st.upload(*host)
    st.forward()
    torch.cuda.synchronize()
    acts = {k: v.interior().cpu().numpy() for k, v in st.out.items() if k != "input"}
    return st.probs.cpu().numpy(), acts
base_p, base_a = run(False, 1, True)
for ov, pdl in ((True, 1), (True, 0), (False, 0)):
    p, a = run(ov, pdl, True)
    diff = [k for k in base_a if not np.array_equal(a[k], base_a[k])]
    print(f"overlap={ov} pdl={pdl}: probs equal {np.array_equal(p, base_p)}; first diffs {diff[:4]}; zero slabs {[k for k in a if not np.any(a[k])][:4]}")
dist.destroy_process_group()
