"""Generate golden vectors by running the REFERENCE pmgflow in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is pure Python/NumPy and has no golden data of its own
(SURVEY 4, 8(c)); its bitwise outputs are platform dependent, so the
fixtures are regenerated here and committed (tests/golden/*.npz).  The
GPU box never reads /root/reference: tests load only these files.

Inputs are the seeded BASELINE-config inputs of paper_2202_09733_b200.cases
(identical arrays to the reference's own harness.isentropic_vortex +
seeded noise).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from pmgflow import mesh as rmesh  # noqa: E402
from pmgflow import newton_krylov as rnk  # noqa: E402
from pmgflow import operators as rops  # noqa: E402
from pmgflow import pmg as rpmg  # noqa: E402
from pmgflow import spatial as rsp  # noqa: E402
from pmgflow import time_integration as rti  # noqa: E402

from paper_2202_09733_b200 import cases  # noqa: E402


def ref_eqn(e):
    return rsp.EquationSpec(kind=e.kind, mach=e.mach, reynolds=e.reynolds, ref_length=e.ref_length,
                            gamma=e.gamma, prandtl=e.prandtl, advection=e.advection, diffusivity=e.diffusivity)


def small_residuals(out):
    """R(q) for every kind x boundary type x a few degrees."""
    meshes = {
        "box4p": rmesh.generate_box(4, 4, 1.0, 1.0, periodic=True),
        "box3ff": rmesh.generate_box(3, 3, 2.0, 1.5),
        "cyl_adiab": rmesh.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3),
        "cyl_slip": rmesh.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3, wall_tag="wall-slip"),
    }
    kinds = {
        "euler": dict(kind="euler", mach=0.3),
        "ns": dict(kind="navier-stokes", mach=0.3, reynolds=200.0),
        "advd": dict(kind="advection-diffusion", advection=(0.7, 0.4), diffusivity=0.02),
    }
    for mname, m in meshes.items():
        for kname, kw in kinds.items():
            for p in (1, 2, 3, 4):
                d = rsp.Discretization(m, p, rsp.EquationSpec(**kw))
                rng = np.random.default_rng(100 + p)
                if kname == "advd":
                    q = rng.standard_normal(d.n_dofs)
                else:
                    q = d.free_stream_field().data * (1 + 0.01 * rng.standard_normal(d.n_dofs))
                out[f"res/{mname}/{kname}/p{p}/q"] = q
                out[f"res/{mname}/{kname}/p{p}/R"] = d.residual(q)


def operators(out):
    for p in range(6):
        b = rops.basis(p)
        out[f"ops/p{p}/D"] = b.diff_matrix
        out[f"ops/p{p}/w"] = b.weights
        out[f"ops/p{p}/eR"] = b.eval_at(np.array([1.0]))[0]
    for pf in range(1, 6):
        for pc in range(pf):
            t = rops.transfer_operators(pf, pc)
            out[f"ops/T{pf}{pc}/gamma"] = t.gamma
            out[f"ops/T{pf}{pc}/pi"] = t.pi


def meshes(out):
    for name, m in {"box4p": rmesh.generate_box(4, 4, 1.0, 1.0, periodic=True),
                    "box3ff": rmesh.generate_box(3, 3, 2.0, 1.5),
                    "cyl": rmesh.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3)}.items():
        out[f"mesh/{name}/interior_faces"] = m.interior_faces
        out[f"mesh/{name}/boundary_faces"] = m.boundary_faces
        g = rmesh.element_geometry(m, 3)
        out[f"mesh/{name}/det"] = g.det
        out[f"mesh/{name}/normals"] = g.face_normals
        out[f"mesh/{name}/face_jac"] = g.face_jac


def blocks_small(out):
    """FD element blocks + inverses, and EJ apply (newton_krylov.py:157-214)."""
    m = rmesh.generate_box(3, 3, 1.0, 1.0, periodic=True)
    eqn = rsp.EquationSpec(kind="navier-stokes", mach=0.3, reynolds=100.0)
    d = rsp.Discretization(m, 2, eqn)
    rng = np.random.default_rng(7)
    q = d.free_stream_field().data * (1 + 0.01 * rng.standard_normal(d.n_dofs))
    bj = rnk.assemble_element_blocks(d, q, 30.0)
    X = rng.standard_normal(d.n_dofs)
    out["blk/q"] = q
    out["blk/blocks"] = bj.blocks[0]
    out["blk/inv"] = bj.inv[0]
    out["blk/X"] = X
    out["blk/Y"] = rnk.ej_apply(bj, X)
    fr = d.freeze(q)
    e = 4
    out["blk/local_e4"] = d.element_residual(e, q[d.offsets[e]:d.offsets[e + 1]].reshape(3, 3, 4) * 1.001, fr)


class GmresLog:
    def __init__(self):
        self.counts = []
        self._orig = rnk.gmres_solve

    def __enter__(self):
        def wrapped(*a, **k):
            x, it, rr = self._orig(*a, **k)
            self.counts.append(it)
            return x, it, rr
        rnk.gmres_solve = wrapped
        return self

    def __exit__(self, *exc):
        rnk.gmres_solve = self._orig


def config1(out):
    c = cases.config(1)
    eqn = ref_eqn(c.eqn)
    m = rmesh.generate_box(16, 16, 10.0, 10.0, periodic=True)
    d = rsp.Discretization(m, 3, eqn)
    q = c.q0
    R0 = d.residual(q)
    rng = np.random.default_rng(11)
    v = rng.standard_normal(d.n_dofs)
    vu = v / np.linalg.norm(v)
    out["c1/q0"] = q
    out["c1/R0"] = R0
    out["c1/v"] = v
    out["c1/Jv"] = rnk.jfnk_matvec(v, q, R0, d.residual, 3.7)
    out["c1/Jvu"] = rnk.jfnk_matvec(vu, q, R0, d.residual, 3.7)
    out["c1/dt"] = np.array(c.dt)
    # pMG preconditioner application at a stage shift
    sch = rti.get_scheme("esdirk2")
    a_ii = float(sch.a[1, 1])
    shift = 1.0 / (a_ii * c.dt) + 1.0 / c.dt
    h = rpmg.PHierarchy.parse("3-2", "2", "ej")
    ctx = rpmg.PmgContext(d, rpmg.PmgPrecondConfig(h, smoother_shift=50.0))
    ctx.prepare(q, shift)
    out["c1/pc_shift"] = np.array(shift)
    out["c1/pc_Y"] = ctx.precondition(vu)
    # one ESDIRK2 step, pMG p{3-2}, smoother_shift 50, dtau_init = dt
    from pmgflow import harness as hz
    cfg = hz.parse_config_text(f"""
case.precond = pmg
pmg.levels = 3-2
pmg.smooth = 2
pmg.smoother_shift = 50
gmres.kdim = 30
gmres.rtol = 1e-3
ptc.dtau_init = {c.dt!r}
ptc.rtol = 1e-4
""")
    for scheme in ("esdirk2", "row4"):
        drv = hz.ImplicitDriver(d, cfg)
        t0 = time.perf_counter()
        with GmresLog() as log:
            sch = rti.get_scheme(scheme)
            if sch.kind == "esdirk":
                qn, info = rti.esdirk_step(q, c.dt, sch, d.residual, drv.solve_stage)
                ptc = [i["iters"] for i in info]
            else:
                Rl = d.residual(q)
                qn, info = rti.row_step(q, c.dt, sch, d.residual, drv.solve_linear(q, Rl))
                ptc = [0] * len(info)
        wall = time.perf_counter() - t0
        out[f"c1/{scheme}/q1"] = qn
        out[f"c1/{scheme}/gmres_counts"] = np.array(log.counts)
        out[f"c1/{scheme}/ptc_iters"] = np.array(ptc)
        out[f"c1/{scheme}/wall_s"] = np.array(wall)
        print(scheme, "gmres per solve", log.counts, "ptc", ptc, f"{wall:.2f}s")


def pmg_solver(out):
    """pmg_solve on a reduced config-3 analogue."""
    c = cases.config(3, nx=4)
    eqn = ref_eqn(c.eqn)
    m = rmesh.generate_box(4, 4, 10.0, 10.0, periodic=True)
    d = rsp.Discretization(m, 4, eqn)
    h = rpmg.PHierarchy.parse("4-3-2-1-0", "2", "ej")
    ctx = rpmg.PmgContext(d, rpmg.PmgPrecondConfig(h, smoother_shift=1e3))
    cfg = rnk.PtcConfig(dtau_init=0.1, dtau_max=1e12, max_iters=6, rtol=1e-10)
    q, st = rpmg.pmg_solve(ctx, c.q0, cfg)
    out["c3/q0"] = c.q0
    out["c3/q"] = q
    out["c3/history"] = np.array(st["history"])


def main():
    out = {}
    operators(out)
    meshes(out)
    small_residuals(out)
    blocks_small(out)
    config1(out)
    pmg_solver(out)
    np.savez_compressed(HERE / "golden.npz", **out)
    size = (HERE / "golden.npz").stat().st_size
    print(f"wrote {len(out)} arrays, {size / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
