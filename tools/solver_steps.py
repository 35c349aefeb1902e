"""Time JFNK-pMG steps on a BASELINE config with solver variants.

    python tools/solver_steps.py CONFIG NSTEPS VARIANT [VARIANT ...]
    VARIANT = scheme:smoothers:smoother_shift[:rk_cfl[:smooth[:stages]]]
              e.g. esdirk3:rk-ej:50:1.5:1-2:0.25/0.5/1  (stages '/'-separated)
    env: NX (mesh override), MAX_PTC, RESTARTS (caps for exploration runs),
         DT_SCALE (multiplies the case's dt), BLOCK_PRECISION (fp64 | fp32),
         DTAU_SCALE (ptc.dtau_init = DTAU_SCALE x dt), PTC_RTOL (default 1e-4)

Prints one JSON line per variant: per-step device wall time (synchronised),
PTC / GMRES iteration counts, peak device memory.  Used for the DESIGN.md
solver tables (config 2 EJ vs RK fine smoothing, config 5 at capacity).
"""
import gc
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2202_09733_b200 import cases  # noqa: E402
from paper_2202_09733_b200 import time_integration as ti  # noqa: E402
from paper_2202_09733_b200.harness import ImplicitDriver  # noqa: E402
from paper_2202_09733_b200.spatial import Discretization  # noqa: E402


def main():
    k, nsteps = int(sys.argv[1]), int(sys.argv[2])
    nx = int(os.environ["NX"]) if os.environ.get("NX") else None
    t0 = time.perf_counter()
    c = cases.config(k, nx=nx)
    if os.environ.get("DT_SCALE"):
        c.dt *= float(os.environ["DT_SCALE"])
    print(json.dumps({"case_built_s": round(time.perf_counter() - t0, 1), "nx": nx, "dt": c.dt}), flush=True)
    d = Discretization(c.mesh, c.p, c.eqn)
    for var in sys.argv[3:]:
        parts = var.split(":")
        scheme, smoothers, shift = parts[0], parts[1], float(parts[2])
        cfl = float(parts[3]) if len(parts) > 3 else 1.5
        smooth = parts[4] if len(parts) > 4 else "2"
        stages = parts[5].replace("/", ",") if len(parts) > 5 else "0.25,0.3333333333333333,0.5,1.0"
        cfg = {"case.precond": "pmg", "pmg.levels": c.levels, "pmg.smooth": smooth, "pmg.smoother": smoothers,
               "pmg.rk.stages": stages,
               "pmg.smoother_shift": shift, "pmg.rk.cfl": cfl, "gmres.kdim": c.kdim, "gmres.rtol": 1e-3,
               "ptc.dtau_init": c.dt * float(os.environ.get("DTAU_SCALE", 1.0)),
               "ptc.rtol": float(os.environ.get("PTC_RTOL", 1e-4)),
               "ptc.max_iters": int(os.environ.get("MAX_PTC", 100)),
               "gmres.max_restarts": int(os.environ.get("RESTARTS", 10)),
               "pmg.block_precision": os.environ.get("BLOCK_PRECISION", "fp64")}
        sch = ti.get_scheme(scheme)
        q = torch.as_tensor(c.q0, device="cuda")
        torch.cuda.reset_peak_memory_stats()
        rec = {"config": k, "variant": var, "dt": c.dt, "n_dofs": d.n_dofs, "steps": []}
        try:
            drv = ImplicitDriver(d, cfg)
            orig = drv.solve_stage

            def logged(prob, q0, orig=orig):
                ts = time.perf_counter()
                qn, stt = orig(prob, q0)
                torch.cuda.synchronize()
                print(json.dumps({"stage_s": round(time.perf_counter() - ts, 3), "ptc": stt["iters"],
                                  "gmres": stt["gmres_iters"], "converged": stt["converged"],
                                  "rel": [round(h[1], 6) for h in stt["history"]][-3:]}), flush=True)
                return qn, stt
            drv.solve_stage = logged
            for st in range(nsteps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                q, info = drv.step(q, c.dt, sch)
                torch.cuda.synchronize()
                el = time.perf_counter() - t0
                rec["steps"].append({"s": round(el, 4),
                                     "ptc": [i.get("iters") for i in info] if sch.kind == "esdirk" else None,
                                     "gmres": [i.get("gmres_iters", i.get("iters")) for i in info]})
                print(json.dumps({"variant": var, "step": st, **rec["steps"][-1]}), flush=True)
        except Exception as exc:
            rec["error"] = f"{type(exc).__name__}: {str(exc)[:300]}"
        rec["peak_gb"] = torch.cuda.max_memory_allocated() / 1e9
        print(json.dumps(rec), flush=True)
        drv = None
        gc.collect()   # drv.solve_stage = logged closes a reference cycle
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
