"""Component-wise device vs oracle on the config-4 wall stretching
(nx x 128 channel, p=3): R, Jv, EJ blocks apply, pMG precondition."""
import sys
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

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ny = int(sys.argv[2]) if len(sys.argv) > 2 else 128
h = 1e-4 * 1.0497 ** np.arange(128)
yn = np.concatenate([[0.0], np.cumsum(h)])
yn = (yn / yn[-1])[: ny + 1]
mesh = generate_channel(nx, ny, nx * 4.0 / 512, yn)
eqn = EquationSpec(kind="navier-stokes", mach=0.2, reynolds=1e4, ref_length=1.0)
xy = solution_point_coords(mesh, 3)
y = xy[..., 1]
u = np.tanh(y / 0.05)
p = np.full_like(y, 1.0 / (eqn.gamma * eqn.mach ** 2))
E = p / (eqn.gamma - 1.0) + 0.5 * u * u
q0 = np.stack([np.ones_like(y), u, 0 * u, E], axis=-1).reshape(-1)
q0 = q0 + 1e-5 * np.random.default_rng(0).uniform(-1, 1, q0.shape)
dt = cases.explicit_dt(mesh, 3, eqn, q0)
sigma = 1.0 / (ti.get_scheme("row4").gamma * dt)
rel = lambda a, b: float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
d = Discretization(mesh, 3, eqn)
o = OracleDisc(mesh, 3, eqn)
q = torch.as_tensor(q0, device="cuda")
R = d.residual(q).cpu().numpy()
Ro = o.residual(q0)
print(f"{nx}x{ny}: M={mesh.n_elements} R rel {rel(R, Ro):.3e}  |R|max {np.abs(Ro).max():.3e}", flush=True)
v = np.random.default_rng(1).standard_normal(q0.size)
v /= np.linalg.norm(v)
Jv = nk.jfnk_matvec(torch.as_tensor(v, device="cuda"), q, torch.as_tensor(Ro, device="cuda"), d.residual, sigma).cpu().numpy()
Jvo = so.jfnk_matvec(v, q0, Ro, o.residual, sigma)
print(f"Jv rel {rel(Jv, Jvo):.3e}", flush=True)
bj = nk.assemble_element_blocks(d, q, sigma + 50.0)
ob = so.assemble_blocks(o, q0, sigma + 50.0)
print(f"EJ apply rel {rel(bj.apply(torch.as_tensor(v, device='cuda')).cpu().numpy(), ob.apply(v)):.3e}", flush=True)
ctx = pmg.PmgContext(d, pmg.PmgPrecondConfig(pmg.PHierarchy.parse("3-2", "2"), smoother_shift=50.0))
ctx.prepare(q, sigma)
octx = so.Pmg(o, "3-2", 2, smoother_shift=50.0)
octx.prepare(q0, sigma)
P = ctx.precondition(torch.as_tensor(v, device="cuda")).cpu().numpy()
Po = octx.precondition(v)
print(f"precondition rel {rel(P, Po):.3e}  |P| {np.abs(Po).max():.3e}  fallbacks dev {getattr(ctx, 'fallbacks', '?')} or {getattr(octx, 'fallbacks', '?')}", flush=True)
