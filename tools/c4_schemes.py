"""Config-4 ROW step at full size for each (scheme, bottom wall, dt factor):
GMRES iterations per stage or the failure.  Usage:
    python tools/c4_schemes.py [nx]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2202_09733_b200 import cases, time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.mesh import generate_channel
from paper_2202_09733_b200.spatial import Discretization

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
c = cases.config(4)
yn = np.unique(c.mesh.nodes[:, 1])
for wall in ("wall-isothermal", "wall-adiabatic"):
    mesh = generate_channel(nx, 128, nx * 4.0 / 512, yn, bottom=wall, top="wall-slip")
    d = Discretization(mesh, 3, c.eqn)
    q0 = torch.as_tensor(c.q0[: d.n_dofs] if nx == 512 else np.tile(c.q0.reshape(128, 512, -1)[:, :nx].reshape(-1), 1),
                         device="cuda")
    for name in ("ros4l", "row4"):
        for f in (1.0, 0.5, 0.25):
            cfg = {"case.precond": "pmg", "pmg.levels": "3-2", "pmg.smooth": "2", "pmg.smoother_shift": 50.0,
                   "gmres.kdim": 60, "gmres.rtol": 1e-3, "gmres.max_restarts": 3}
            t0 = time.perf_counter()
            try:
                _, info = ImplicitDriver(d, cfg).step(q0, f * c.dt, ti.get_scheme(name))
                res = [i["iters"] for i in info]
            except Exception as exc:
                res = str(exc)[:90]
            torch.cuda.synchronize()
            print(f"{wall:16s} {name:6s} dt x{f:5.2f}: {res}  {time.perf_counter() - t0:.2f}s", flush=True)
