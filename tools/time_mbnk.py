"""MBNK pieces at scale: block-sparse assembly, ILU0 factor / apply, SpMV
on config 2's coarse level (p=2, 65536 elements), then one ESDIRK2 step
with EJ on the fine and MBNK on the coarse level."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, newton_krylov as nk, pmg, time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.spatial import Discretization

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
c = cases.config(2, nx=nx)
dc = Discretization(c.mesh, 2, c.eqn)
q2 = torch.as_tensor(cases.config(2, nx=nx).q0, device="cuda")
ctx0 = pmg.PmgContext(Discretization(c.mesh, 4, c.eqn), pmg.PmgPrecondConfig(pmg.PHierarchy.parse("4-2")))
qc = ctx0.tables[0].restrict(q2)
def tm(fn, n=1):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n, r
t, _ = tm(lambda: nk.sparse_pattern(dc))
print(f"pattern (host, once per mesh): {t*1e3:.0f} ms; levels lo {len(nk.sparse_pattern(dc).lo_ptr)-1} up {len(nk.sparse_pattern(dc).up_ptr)-1}", flush=True)
t, A = tm(lambda: nk.assemble_sparse_blocks(dc, qc, 40.0))
print(f"sparse assembly p=2 M={c.mesh.n_elements}: {t*1e3:.1f} ms, nnz {A.pattern.nnz}", flush=True)
t, F = tm(lambda: nk.ilu0_factor(A))
print(f"ILU0 factor: {t*1e3:.1f} ms", flush=True)
v = torch.randn(dc.n_dofs, dtype=torch.float64, device="cuda")
t, _ = tm(lambda: nk.ilu0_apply(F, v), 5)
print(f"ILU0 apply: {t*1e3:.2f} ms", flush=True)
t, _ = tm(lambda: A.matvec(v), 20)
print(f"SpMV: {t*1e3:.3f} ms", flush=True)
del A, F
d = Discretization(c.mesh, c.p, c.eqn)
cfg = {"case.precond": "pmg", "pmg.levels": "4-2", "pmg.smooth": "2", "pmg.smoother": "ej-mbnk",
       "pmg.smoother_shift": c.extra["smoother_shift"], "gmres.kdim": 30, "gmres.rtol": 1e-3,
       "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4}
s = ti.get_scheme("esdirk2")
for rep in range(2 if "--step" in sys.argv else 0):
    drv = ImplicitDriver(d, cfg)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    try:
        q1, info = drv.step(q2, c.dt, s)
        res = [(i["iters"], i["gmres_iters"]) for i in info]
    except Exception as exc:
        res = str(exc)[:200]
    torch.cuda.synchronize()
    print(f"ESDIRK2 step config2@{nx} ej-mbnk: {time.perf_counter()-t0:.2f} s {res}", flush=True)
