"""Quick device timing of R / Jv at a BASELINE config (diagnostic)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2202_09733_b200 import cases, _lib
from paper_2202_09733_b200.spatial import Discretization

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = cases.config(k)
d = Discretization(c.mesh, c.p, c.eqn)
q = torch.as_tensor(c.q0, device="cuda")
X = torch.randn_like(q)
R = d.residual(q)
out = torch.empty_like(q)
for mode, name in ((_lib.EPI_R, "R"), (_lib.EPI_JV, "Jv")):
    for _ in range(3):
        d.eval(q, mode, out, X=X, eps=1e-6, s=1.0, R0=R)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    ev0.record()
    for _ in range(reps):
        d.eval(q, mode, out, X=X, eps=1e-6, s=1.0, R0=R)
    ev1.record(); torch.cuda.synchronize()
    t = ev0.elapsed_time(ev1) / reps * 1e-3
    print(f"config{k} {name}: {t*1e6:.1f} us  {d.n_dofs/t/1e9:.2f} GDoF/s  ({d.n_dofs} DoF)")
