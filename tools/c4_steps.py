"""Config-4 multi-step runs per (bottom wall, scheme, dt factor): GMRES per
stage per step, or the step where it fails.
    python tools/c4_steps.py NSTEPS [nx]"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2202_09733_b200 import cases, time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.mesh import generate_channel
from paper_2202_09733_b200.spatial import Discretization

nsteps = int(sys.argv[1])
nx = int(sys.argv[2]) if len(sys.argv) > 2 else 512
c = cases.config(4)
yn = np.unique(c.mesh.nodes[:, 1])
for wall in ("wall-isothermal", "wall-adiabatic"):
    mesh = generate_channel(nx, 128, nx * 4.0 / 512, yn, bottom=wall, top="wall-slip")
    d = Discretization(mesh, 3, c.eqn)
    q0 = torch.as_tensor(c.q0.reshape(128, 512, -1)[:, :nx].reshape(-1).copy(), device="cuda")
    for name, f in (("ros4l", 1.0), ("ros4l", 0.5), ("row4", 2.0), ("row4", 1.0)):
        cfg = {"case.precond": "pmg", "pmg.levels": "3-2", "pmg.smooth": "2", "pmg.smoother_shift": 50.0,
               "gmres.kdim": 60, "gmres.rtol": 1e-3, "gmres.max_restarts": 3}
        drv = ImplicitDriver(d, cfg)
        q, hist, err = q0.clone(), [], None
        t0 = time.perf_counter()
        for s in range(nsteps):
            try:
                q, info = drv.step(q, f * c.dt, ti.get_scheme(name))
                hist.append(max(i["iters"] for i in info))
            except Exception as exc:
                err = f"step {s}: {str(exc)[:80]}"
                break
        torch.cuda.synchronize()
        print(json.dumps({"wall": wall, "scheme": name, "dt_factor_vs_case": f, "steps_done": len(hist),
                          "max_gmres_per_step": hist, "error": err, "s": round(time.perf_counter() - t0, 2)}),
              flush=True)
