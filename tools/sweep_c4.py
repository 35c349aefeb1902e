"""Find EJ smoother shifts for which the full config-4 ROW4 step converges
(stretched wall cells: viscous spectral radius ~ mu (p+1)^4 / h0^2)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.spatial import Discretization

nx = int(sys.argv[3]) if len(sys.argv) > 3 else None
c = cases.config(4, nx=nx)
d = Discretization(c.mesh, c.p, c.eqn)
q = torch.as_tensor(c.q0, device="cuda")
shifts = [float(s) for s in sys.argv[1].split(",")]
restarts = int(sys.argv[2]) if len(sys.argv) > 2 else 2
print(f"config4 nx={nx}: dt {c.dt:.3e}, h_min {c.mesh.h_min:.3e}, n_dofs {d.n_dofs}", flush=True)
for sh in shifts:
    for levels in (c.levels,):
        cfg = {"case.precond": "pmg", "pmg.levels": levels, "pmg.smooth": "2", "pmg.smoother_shift": sh,
               "gmres.kdim": c.kdim, "gmres.rtol": 1e-3, "gmres.max_restarts": restarts}
        drv = ImplicitDriver(d, cfg)
        t0 = time.perf_counter()
        try:
            q1, info = drv.step(q, c.dt, ti.get_scheme("row4"))
            res = [(i["iters"], round(float(i.get("relres", 0)), 5)) for i in info]
        except Exception as e:
            res = str(e)[:200]
        torch.cuda.synchronize()
        print(f"shift {sh:9.1f} levels {levels}: {time.perf_counter() - t0:6.2f}s  {res}", flush=True)
