"""Golden vectors for the MBNK smoother path, made by
running the REFERENCE pmgflow in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_mbnk.py

Block-sparse FD Jacobians (assemble_sparse_blocks), their block ILU0
factors, SparseBlockMatrix.matvec and ilu0_apply on small meshes covering
periodic (incl. a 2x2 mesh whose element pairs meet through two faces),
far-field and adiabatic-wall boundaries; MBNK-smoothed pMG precondition
calls on reduced config 1; a pmg_solve run with switch_after.  Written to
tests/golden/golden_mbnk.npz (the GPU box only reads that file).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

from pmgflow import mesh as rmesh  # noqa: E402
from pmgflow import newton_krylov as rnk  # noqa: E402
from pmgflow import pmg as rpmg  # noqa: E402
from pmgflow import spatial as rsp  # noqa: E402
from pmgflow import time_integration as rti  # noqa: E402

from paper_2202_09733_b200 import cases  # noqa: E402

SPARSE_CASES = {
    "box3p_ns1": (lambda: rmesh.generate_box(3, 3, 1.0, 1.0, periodic=True),
                  dict(kind="navier-stokes", mach=0.3, reynolds=100.0), 1),
    "box2p_ns1": (lambda: rmesh.generate_box(2, 2, 1.0, 1.0, periodic=True),
                  dict(kind="navier-stokes", mach=0.3, reynolds=100.0), 1),
    "cyl_ns1": (lambda: rmesh.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3),
                dict(kind="navier-stokes", mach=0.3, reynolds=200.0), 1),
    "box3ff_euler2": (lambda: rmesh.generate_box(3, 3, 2.0, 1.5),
                      dict(kind="euler", mach=0.3), 2),
}


def ref_eqn(e):
    return rsp.EquationSpec(kind=e.kind, mach=e.mach, reynolds=e.reynolds, ref_length=e.ref_length,
                            gamma=e.gamma, prandtl=e.prandtl, advection=e.advection, diffusivity=e.diffusivity)


def sparse(out):
    for name, (mk, kw, p) in SPARSE_CASES.items():
        d = rsp.Discretization(mk(), p, rsp.EquationSpec(**kw))
        rng = np.random.default_rng(11)
        q = d.free_stream_field().data * (1 + 0.01 * rng.standard_normal(d.n_dofs))
        S = rnk.assemble_sparse_blocks(d, q, 40.0)
        fac = rnk.ilu0_factor(S)
        X = rng.standard_normal(d.n_dofs)
        out[f"sp/{name}/q"] = q
        out[f"sp/{name}/indptr"] = np.asarray(S.indptr)
        out[f"sp/{name}/indices"] = np.asarray(S.indices)
        out[f"sp/{name}/blocks"] = np.stack(S.blocks)
        out[f"sp/{name}/lu"] = np.stack(fac.pattern.blocks)
        out[f"sp/{name}/dinv"] = np.stack(fac.diag_inv)
        out[f"sp/{name}/X"] = X
        out[f"sp/{name}/AX"] = S.matvec(X, d.offsets)
        out[f"sp/{name}/iluX"] = rnk.ilu0_apply(fac, X, d.offsets)
        print(name, "nnz", len(S.indices))


def mbnk_precondition(out):
    c = cases.config(1, nx=4)
    d = rsp.Discretization(rmesh.generate_box(4, 4, 10.0, 10.0, periodic=True), 3, ref_eqn(c.eqn))
    q = c.q0
    v = np.random.default_rng(3).standard_normal(d.n_dofs)
    v /= np.linalg.norm(v)
    shift = 1.0 / (float(rti.get_scheme("esdirk2").a[1, 1]) * c.dt) + 1.0 / c.dt
    out["mb/q"] = q
    out["mb/v"] = v
    out["mb/shift"] = np.array(shift)
    for kinds in ("mbnk", "ej-mbnk"):
        h = rpmg.PHierarchy.parse("3-2", "1", kinds)
        ctx = rpmg.PmgContext(d, rpmg.PmgPrecondConfig(h, smoother_shift=50.0))
        ctx.prepare(q, shift)
        out[f"mb/{kinds}/Y"] = ctx.precondition(v)
        print("precondition", kinds, "done")


def switch_after(out):
    # config-1 physics (Ma 0.5): the low-Mach config 3 amplifies FD noise too
    # much for a tight history comparison
    c = cases.config(1, nx=4)
    d = rsp.Discretization(rmesh.generate_box(4, 4, 10.0, 10.0, periodic=True), 3, ref_eqn(c.eqn))
    h = rpmg.PHierarchy.parse("3-2", "1", "ej", switch_after=1)
    ctx = rpmg.PmgContext(d, rpmg.PmgPrecondConfig(h, smoother_shift=50.0))
    cfg = rnk.PtcConfig(dtau_init=0.05, dtau_max=1e12, max_iters=3, rtol=1e-12)
    q, st = rpmg.pmg_solve(ctx, c.q0, cfg)
    out["sw/q0"] = c.q0
    out["sw/q"] = q
    out["sw/history"] = np.array(st["history"])
    print("switch_after history", st["history"])


def main():
    out = {}
    sparse(out)
    mbnk_precondition(out)
    switch_after(out)
    np.savez_compressed(HERE / "golden_mbnk.npz", **out)
    print(f"wrote {len(out)} arrays, {(HERE / 'golden_mbnk.npz').stat().st_size / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
