import sys, numpy as np, torch, json
sys.path.insert(0, '.')
from paper_2202_09733_b200 import cases, time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.spatial import Discretization
c = cases.config(2, nx=48)
s = ti.get_scheme("esdirk3")
for path in ("rect", "general"):
    d = Discretization(c.mesh, c.p, c.eqn)
    d.residual_path(path)
    cfg = {"case.precond": "pmg", "pmg.levels": c.levels, "pmg.smooth": "2", "pmg.smoother_shift": c.extra["smoother_shift"],
           "gmres.kdim": 30, "gmres.rtol": 1e-3, "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4}
    q_d, info = ImplicitDriver(d, cfg).step(torch.as_tensor(c.q0, device="cuda"), c.dt, s)
    print(path, [(i["iters"], i["gmres_iters"], i.get("gmres_per_iter")) for i in info])
    np.save(f"gpurun_out/q48_{path}.npy", q_d.cpu().numpy())
