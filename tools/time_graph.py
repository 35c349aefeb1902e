"""Step time with precondition() replayed as a CUDA graph (pmg.graph = on) against
the eager launch sequence (off): python tools/time_graph.py [config[:nx]...] (default 1 2)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2202_09733_b200 import cases  # noqa: E402
from paper_2202_09733_b200 import time_integration as ti  # noqa: E402
from paper_2202_09733_b200.harness import ImplicitDriver  # noqa: E402
from paper_2202_09733_b200.spatial import Discretization  # noqa: E402

import os  # noqa: E402

for arg in sys.argv[1:] or ["1", "2"]:
    k, _, nx = arg.partition(":")   # "1:64" = config 1's physics on a 64 x 64 mesh
    k = int(k)
    c = cases.config(k, nx=int(nx) if nx else None)
    d = Discretization(c.mesh, c.p, c.eqn)
    s = ti.get_scheme(c.scheme)
    rec = {"config": arg, "n_dofs": d.n_dofs, "scheme": c.scheme}
    for g in ("off", "on", "off", "on"):
        cfg = {"case.precond": "pmg", "pmg.levels": c.levels, "pmg.smooth": "2",
               "pmg.smoother_shift": c.extra.get("smoother_shift", 50.0), "gmres.kdim": c.kdim, "gmres.rtol": 1e-3,
               "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4, "pmg.graph": g}
        drv = ImplicitDriver(d, cfg)
        q = torch.as_tensor(c.q0, device="cuda")
        drv.step(q, c.dt, s)   # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q1, info = drv.step(q, c.dt, s)
        torch.cuda.synchronize()
        rec.setdefault(g, []).append({"step_s": round(time.perf_counter() - t0, 4),
                                      "gmres": [i.get("gmres_iters", i.get("iters")) for i in info],
                                      "replays": drv.ctx.graph_replays})
    print(json.dumps(rec), flush=True)
