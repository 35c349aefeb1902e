"""Config 3 (low-Mach steady, 128^2, p=4): the nonlinear pMG solver
(pmg_solve, pmg.py:308-374) over p{4-3-2-1-0} run toward BASELINE's
10-order residual drop.  One JSON line per variant:
    python tools/c3_converge.py MAX_ITERS VARIANT [VARIANT ...]
    VARIANT = smoothers:smoother_shift:dtau_init:refresh_every[:rk_cfl]
    e.g. rk-rk-rk-rk-ej:1000:0.1:10"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, newton_krylov as nk, pmg
from paper_2202_09733_b200.spatial import Discretization

max_iters = int(sys.argv[1])
c = cases.config(3)
d = Discretization(c.mesh, c.p, c.eqn)
q0 = torch.as_tensor(c.q0, device="cuda")
for var in sys.argv[2:]:
    parts = var.split(":")
    sm, shift, dtau, refresh = parts[0], float(parts[1]), float(parts[2]), int(parts[3])
    cfl = float(parts[4]) if len(parts) > 4 else 1.5
    hier = pmg.PHierarchy.parse(c.levels, "2", sm)
    ctx = pmg.PmgContext(d, pmg.PmgPrecondConfig(hier, smoother_shift=shift, rk_cfl=cfl))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        q, st = pmg.pmg_solve(ctx, q0, nk.PtcConfig(dtau_init=dtau, max_iters=max_iters, rtol=1e-10,
                                                    refresh_every=refresh))
        torch.cuda.synchronize()
        h = st["history"]
        rec = {"variant": var, "iters": st["iters"], "converged": st["converged"], "aborted": st["aborted"],
               "s": round(time.perf_counter() - t0, 3), "final_rel": h[-1][1],
               "rel_every_10": [float(f"{x[1]:.3e}") for x in h[::10]], "dtau_final": h[-1][2]}
    except Exception as exc:
        rec = {"variant": var, "error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    print(json.dumps(rec), flush=True)
    del ctx
    torch.cuda.empty_cache()
