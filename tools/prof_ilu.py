import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, newton_krylov as nk
from paper_2202_09733_b200.spatial import Discretization
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 64
c = cases.config(2, nx=nx)
dc = Discretization(c.mesh, 2, c.eqn)
q = torch.ones(dc.n_dofs, dtype=torch.float64, device="cuda")
q.view(-1, 4)[:, 3] = 7.64
A = nk.assemble_sparse_blocks(dc, q, 40.0)
F = nk.ilu0_factor(A)
v = torch.randn(dc.n_dofs, dtype=torch.float64, device="cuda")
nk.ilu0_apply(F, v); torch.cuda.synchronize()
t0 = time.perf_counter(); nk.ilu0_apply(F, v); torch.cuda.synchronize()
print(f"apply {nx}: {(time.perf_counter()-t0)*1e3:.2f} ms, levels {len(F.pattern.pattern.lo_ptr)-1}")
