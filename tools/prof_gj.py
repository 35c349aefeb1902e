"""Small-grid driver for ncu captures of k_blocks / k_gj_inverse at p=4."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import _lib, cases
from paper_2202_09733_b200.spatial import Discretization
from paper_2202_09733_b200.vec import stream

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = cases.config(2, nx=nx)
d = Discretization(c.mesh, c.p, c.eqn)
q = torch.as_tensor(c.q0, device="cuda")
M, sz = c.mesh.n_elements, d.elem_size
B = torch.empty((M, sz, sz), dtype=torch.float64, device="cuda")
X = torch.empty_like(B)
perm = torch.empty((M, 2 * sz), dtype=torch.uint8, device="cuda")
lib = _lib.load()
for _ in range(reps):
    lib.pmgb_blocks_assemble(d._h, q.data_ptr(), 60.0, 1e-6, B.data_ptr(), None, None, stream())
    lib.pmgb_blocks_invert(M, sz, B.data_ptr(), X.data_ptr(), perm.data_ptr(), stream())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
lib.pmgb_blocks_invert(M, sz, B.data_ptr(), X.data_ptr(), perm.data_ptr(), stream())
e1.record(); e1.synchronize()
print(f"invert {M} blocks of {sz}: {e0.elapsed_time(e1)*1e3:.1f} us")
