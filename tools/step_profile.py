"""One ESDIRK2 JFNK-pMG step at a BASELINE config (after a warm-up step).

    python tools/step_profile.py [config] [nx]
Under `ncu --metrics gpu__time_duration.sum --csv` the launch list gives the
per-kernel-type device time; without ncu it prints the wall time."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.spatial import Discretization
from paper_2202_09733_b200.vec import launch_count

pos = [a for a in sys.argv[1:] if not a.startswith("--")]
k = int(pos[0]) if pos else 2
nx = int(pos[1]) if len(pos) > 1 else None
warm = "--no-warm" not in sys.argv
c = cases.config(k, nx=nx)
d = Discretization(c.mesh, c.p, c.eqn)
cfg = {"case.precond": "pmg", "pmg.levels": c.levels, "pmg.smooth": "2",
       "pmg.smoother_shift": c.extra["smoother_shift"], "gmres.kdim": c.kdim, "gmres.rtol": 1e-3,
       "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4,
       "pmg.block_precision": "fp32" if "--fp32" in sys.argv else "fp64"}
q = torch.as_tensor(c.q0, device="cuda")
sch = ti.get_scheme(c.scheme if "--case-scheme" in sys.argv else "esdirk2")
if warm:
    ImplicitDriver(d, cfg).step(q, c.dt, sch)
torch.cuda.synchronize()
drv = ImplicitDriver(d, cfg)  # coarse levels built outside the timed step
torch.cuda.synchronize()
l0 = launch_count()
t0 = time.perf_counter()
q1, info = drv.step(q, c.dt, sch)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"config{k}: step {wall * 1e3:.1f} ms, {launch_count() - l0} launches, "
      f"ptc {[i['iters'] for i in info]}, gmres {[i['gmres_iters'] for i in info]}")
if "--cprofile" in sys.argv:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    torch.cuda.synchronize()
    pr.enable()
    ImplicitDriver(d, cfg).step(q, c.dt, sch)
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)
    st.sort_stats("cumulative").print_stats(40)
