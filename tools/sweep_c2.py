"""Find EJ smoother shifts for which the config-2 ESDIRK2 stage converges."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, newton_krylov as nk, time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.spatial import Discretization

c = cases.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
d = Discretization(c.mesh, c.p, c.eqn)
q = torch.as_tensor(c.q0, device="cuda")
shifts = [float(s) for s in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["100", "200", "500", "1000"])]
cfls = [float(s) for s in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["50"])]
from paper_2202_09733_b200.cases import explicit_dt
dt_conv = explicit_dt(c.mesh, c.p, c.eqn, c.q0)
for cfl in cfls:
  c.dt = cfl * dt_conv
  for sh in shifts:
    for levels in (c.levels,):
        cfg = {"case.precond": "pmg", "pmg.levels": levels, "pmg.smooth": "2", "pmg.smoother_shift": sh,
               "gmres.kdim": c.kdim, "gmres.rtol": 1e-3, "gmres.max_restarts": int(sys.argv[4]) if len(sys.argv) > 4 else 2,
               "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4, "ptc.max_iters": 8}
        drv = ImplicitDriver(d, cfg)
        t0 = time.perf_counter()
        try:
            q1, info = drv.step(q, c.dt, ti.get_scheme("esdirk2"))
            res = [(i["iters"], i["gmres_iters"], i["converged"]) for i in info]
        except Exception as e:
            res = str(e)[:160]
        torch.cuda.synchronize()
        print(f"cfl {cfl:5.1f} shift {sh:7.1f} levels {levels}: {time.perf_counter() - t0:6.2f}s  {res}", flush=True)
