import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import os
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np, torch
from oracle import solver_oracle as so
from paper_2202_09733_b200 import time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
import test_gpu_solver as T
c, o, d = T._c2_small(16)
s = ti.get_scheme("esdirk2")
cfg = {"case.precond": "pmg", "pmg.levels": "4-2", "pmg.smooth": "2", "pmg.smoother_shift": 50.0,
       "gmres.kdim": 30, "gmres.rtol": 1e-3, "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4}
res = []
for rep in range(2):
    q_d, info = ImplicitDriver(d, cfg).step(T.t(c.q0), c.dt, s)
    res.append((q_d.cpu().numpy(), [(i["iters"], i["gmres_iters"]) for i in info]))
print("device runs bitwise equal:", np.array_equal(res[0][0], res[1][0]), res[0][1], res[1][1])
ores = []
for rep in range(2):
    drv_o = so.Driver(o, "pmg", "4-2", 2, smoother_shift=50.0, gmres_rtol=1e-3, dtau_init=c.dt)
    q_o = drv_o.esdirk_step(c.q0, c.dt, s.a, s.b)
    ores.append((q_o, [(r[1], r[2]) for r in drv_o.records]))
print("oracle runs bitwise equal:", np.array_equal(ores[0][0], ores[1][0]), ores[0][1], ores[1][1])
print("device vs oracle rel:", np.max(np.abs(res[0][0] - ores[0][0])) / np.max(np.abs(ores[0][0])))
