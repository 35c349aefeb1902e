"""ESDIRK2 step with EJ fine / MBNK coarse smoothing at reduced config 2:
device vs oracle (does the algorithm converge here?)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import solver_oracle as so
from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import cases, time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.spatial import Discretization
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 16
shift = float(sys.argv[2]) if len(sys.argv) > 2 else 5000.0
c = cases.config(2, nx=nx)
d = Discretization(c.mesh, c.p, c.eqn)
s = ti.get_scheme("esdirk2")
cfg = {"case.precond": "pmg", "pmg.levels": "4-2", "pmg.smooth": "2", "pmg.smoother": "ej-mbnk",
       "pmg.smoother_shift": shift, "gmres.kdim": 30, "gmres.rtol": 1e-3, "ptc.dtau_init": c.dt,
       "ptc.rtol": 1e-4, "ptc.max_iters": 8}
t0 = time.perf_counter()
try:
    q1, info = ImplicitDriver(d, cfg).step(torch.as_tensor(c.q0, device="cuda"), c.dt, s)
    print("device", [(i["iters"], i["gmres_iters"]) for i in info], f"{time.perf_counter()-t0:.1f}s", flush=True)
except Exception as e:
    print("device failed:", str(e)[:300], flush=True)
if "--oracle" in sys.argv:
    o = OracleDisc(c.mesh, c.p, c.eqn)
    drv = so.Driver(o, "pmg", "4-2", 2, smoother_shift=shift, gmres_rtol=1e-3, dtau_init=c.dt, max_iters=8)
    drv.ctx = so.Pmg(o, "4-2", 2, smoother_shift=shift, smoother="ej-mbnk")
    t0 = time.perf_counter()
    try:
        drv.esdirk_step(c.q0, c.dt, s.a, s.b)
        print("oracle", [(r[1], r[2]) for r in drv.records], f"{time.perf_counter()-t0:.1f}s")
    except Exception as e:
        print("oracle failed:", str(e)[:300], [(r[1], r[2]) for r in drv.records])
