"""Config-4 wall stretching (h0 = 1e-4, ratio 1.0497, 128 wall-normal cells)
on a narrow x-periodic channel (nx cells over Lx = nx * 4/512, the full
config's dx): first ROW4 linear solve, GMRES(60) without restart, pMG 3-2,
on the device and in the CPU oracle -- the relative-residual histories
show whether a stall is the algorithm's or the device's."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from oracle import solver_oracle as so
from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import cases, newton_krylov as nk, pmg, time_integration as ti
from paper_2202_09733_b200.equation import EquationSpec
from paper_2202_09733_b200.mesh import generate_channel, solution_point_coords
from paper_2202_09733_b200.spatial import Discretization

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 16
shift = float(sys.argv[2]) if len(sys.argv) > 2 else 50.0
kdim = int(sys.argv[3]) if len(sys.argv) > 3 else 60
cfl = float(sys.argv[4]) if len(sys.argv) > 4 and not sys.argv[4].startswith("--") else 10.0
ny = 128
h = 1e-4 * 1.0497 ** np.arange(ny)
yn = np.concatenate([[0.0], np.cumsum(h)])
yn = yn / yn[-1]
mesh = generate_channel(nx, ny, nx * 4.0 / 512, yn)
eqn = EquationSpec(kind="navier-stokes", mach=0.2, reynolds=1e4, ref_length=1.0)
xy = solution_point_coords(mesh, 3)
y = xy[..., 1]
u = np.tanh(y / 0.05)
rho = np.ones_like(y)
p = np.full_like(y, 1.0 / (eqn.gamma * eqn.mach ** 2))
E = p / (eqn.gamma - 1.0) + 0.5 * rho * u * u
q0 = np.stack([rho, rho * u, 0 * u, E], axis=-1).reshape(-1)
q0 = q0 + 1e-5 * np.random.default_rng(0).uniform(-1, 1, q0.shape)
dt = cfl * cases.explicit_dt(mesh, 3, eqn, q0)
s = ti.get_scheme("row4")
sigma = 1.0 / (s.gamma * dt)
print(f"narrow config-4 channel {nx}x{ny}: {q0.size} DoF, dt {dt:.3e}, sigma {sigma:.3e}, shift {shift}")

d = Discretization(mesh, 3, eqn)
q = torch.as_tensor(q0, device="cuda")
R = d.residual(q)
ctx = pmg.PmgContext(d, pmg.PmgPrecondConfig(pmg.PHierarchy.parse("3-2", "2"), smoother_shift=shift))
ctx.prepare(q, sigma)
hist_d = []
def mv(v):
    return nk.jfnk_matvec(v, q, R, d.residual, sigma, check_zero=False, sync=False)
t0 = time.perf_counter()
KDS = [int(a) for a in next((x[6:] for x in sys.argv if x.startswith("--kds=")), "1,5,10,20,40,%d" % kdim).split(",")]
for kd in (KDS if "--restarts" not in sys.argv else (kdim,)):
    mr = 10 if "--restarts" in sys.argv else 1
    x, it, rr = nk.gmres_solve(mv, R, nk.KrylovConfig(kdim=kd, max_restarts=mr, rtol=1e-3 if mr > 1 else 1e-12),
                               precond=ctx.precondition)
    hist_d.append((it, rr))
print("device  (iters, relres):", [(i, f"{r:.4e}") for i, r in hist_d], f"{time.perf_counter() - t0:.1f}s", flush=True)

if "--oracle" in sys.argv:
    o = OracleDisc(mesh, 3, eqn)
    Ro = o.residual(q0)
    octx = so.Pmg(o, "3-2", 2, smoother_shift=shift)
    t0 = time.perf_counter()
    octx.prepare(q0, sigma)
    hist_o = []
    for kd in KDS:
        x, it, rr = so.gmres_solve(lambda v: so.jfnk_matvec(v, q0, Ro, o.residual, sigma), Ro,
                                   kdim=kd, max_restarts=1, rtol=1e-12, precond=octx.precondition)
        hist_o.append((it, rr))
    print("oracle  (iters, relres):", [(i, f"{r:.4e}") for i, r in hist_o], f"{time.perf_counter() - t0:.1f}s")
