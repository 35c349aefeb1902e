"""Device MBNK path through the C ABI against the reference's goldens
(tests/golden/make_golden_mbnk.py) and the oracle: block-sparse FD
Jacobian (element + coupling blocks), block SpMV, block ILU0 factor and
apply, MBNK-smoothed pMG, switch_after.  FD blocks carry the reference's
own FD noise (R rounding x 1/eps), hence ~1e-7-of-scale tolerances."""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2202_09733_b200 import cases, mesh as mm, newton_krylov as nk
from paper_2202_09733_b200.equation import EquationSpec
from paper_2202_09733_b200.spatial import Discretization

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).parent / "golden" / "golden_mbnk.npz")

SPARSE_CASES = {
    "box3p_ns1": (lambda: mm.generate_box(3, 3, 1.0, 1.0, periodic=True),
                  dict(kind="navier-stokes", mach=0.3, reynolds=100.0), 1),
    "box2p_ns1": (lambda: mm.generate_box(2, 2, 1.0, 1.0, periodic=True),
                  dict(kind="navier-stokes", mach=0.3, reynolds=100.0), 1),
    "cyl_ns1": (lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3),
                dict(kind="navier-stokes", mach=0.3, reynolds=200.0), 1),
    "box3ff_euler2": (lambda: mm.generate_box(3, 3, 2.0, 1.5), dict(kind="euler", mach=0.3), 2),
}


def scaled(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def t(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


@pytest.mark.parametrize("name", list(SPARSE_CASES))
def test_sparse_blocks_match_reference(cuda, name):
    mk, kw, p = SPARSE_CASES[name]
    d = Discretization(mk(), p, EquationSpec(**kw))
    pre = f"sp/{name}/"
    A = nk.assemble_sparse_blocks(d, t(G[pre + "q"]), 40.0)
    assert np.array_equal(A.indptr, G[pre + "indptr"]) and np.array_equal(A.indices, G[pre + "indices"])
    assert scaled(A.blocks, G[pre + "blocks"]) <= 1e-7
    assert scaled(A.matvec(t(G[pre + "X"])), G[pre + "AX"]) <= 1e-7


@pytest.mark.parametrize("name", list(SPARSE_CASES))
def test_ilu0_factor_and_apply_match_reference(cuda, name):
    mk, kw, p = SPARSE_CASES[name]
    d = Discretization(mk(), p, EquationSpec(**kw))
    pre = f"sp/{name}/"
    A = nk.assemble_sparse_blocks(d, t(G[pre + "q"]), 40.0)
    fac = nk.ilu0_factor(A)
    assert scaled(fac.pattern.blocks, G[pre + "lu"]) <= 1e-6
    assert scaled(fac.diag_inv, G[pre + "dinv"]) <= 1e-6
    assert scaled(nk.ilu0_apply(fac, t(G[pre + "X"])), G[pre + "iluX"]) <= 1e-6


@pytest.mark.parametrize("kinds", ["mbnk", "ej-mbnk"])
def test_mbnk_precondition_matches_reference(cuda, kinds):
    from paper_2202_09733_b200 import pmg
    c = cases.config(1, nx=4)
    d = Discretization(c.mesh, 3, c.eqn)
    ctx = pmg.PmgContext(d, pmg.PmgPrecondConfig(pmg.PHierarchy.parse("3-2", "1", kinds), smoother_shift=50.0))
    ctx.prepare(t(G["mb/q"]), float(G["mb/shift"]))
    assert scaled(ctx.precondition(t(G["mb/v"])), G[f"mb/{kinds}/Y"]) <= 1e-6


def test_switch_after_pmg_solve_matches_reference(cuda):
    from paper_2202_09733_b200 import pmg
    c = cases.config(1, nx=4)
    d = Discretization(c.mesh, 3, c.eqn)
    h = pmg.PHierarchy.parse("3-2", "1", "ej", switch_after=1)
    ctx = pmg.PmgContext(d, pmg.PmgPrecondConfig(h, smoother_shift=50.0))
    q, st = pmg.pmg_solve(ctx, t(G["sw/q0"]), nk.PtcConfig(dtau_init=0.05, max_iters=3, rtol=1e-12))
    hist, ref = np.array(st["history"]), G["sw/history"]
    assert hist.shape == ref.shape
    assert np.allclose(hist[:, 1], ref[:, 1], rtol=1e-5)
    assert scaled(q, G["sw/q"]) <= 1e-7


def test_mbnk_driver_step_matches_oracle(cuda):
    # an ESDIRK2 step with MBNK smoothing on the coarse level, device vs oracle
    from oracle import solver_oracle as so
    from oracle.fr_oracle import OracleDisc
    from paper_2202_09733_b200 import time_integration as ti
    from paper_2202_09733_b200.harness import ImplicitDriver
    c = cases.config(1, nx=4)
    d = Discretization(c.mesh, 3, c.eqn)
    o = OracleDisc(c.mesh, 3, c.eqn)
    cfg = {"case.precond": "pmg", "pmg.levels": "3-2", "pmg.smooth": "1", "pmg.smoother": "ej-mbnk",
           "pmg.smoother_shift": 50.0, "gmres.rtol": 1e-3, "ptc.dtau_init": c.dt}
    s = ti.get_scheme("esdirk2")
    q1, info = ImplicitDriver(d, cfg).step(t(c.q0), c.dt, s)
    drv = so.Driver(o, "pmg", "3-2", 1, smoother_shift=50.0, gmres_rtol=1e-3, dtau_init=c.dt)
    drv.ctx = so.Pmg(o, "3-2", 1, smoother_shift=50.0, smoother="ej-mbnk")
    q1_o = drv.esdirk_step(c.q0, c.dt, s.a, s.b)
    assert [i["iters"] for i in info] == [r[1] for r in drv.records]
    assert scaled(q1, q1_o) <= 1e-7


@pytest.mark.parametrize("name", list(SPARSE_CASES))
def test_ilu0_fused_apply_is_bitwise_the_level_path(cuda, name):
    mk, kw, p = SPARSE_CASES[name]
    d = Discretization(mk(), p, EquationSpec(**kw))
    pre = f"sp/{name}/"
    fac = nk.ilu0_factor(nk.assemble_sparse_blocks(d, t(G[pre + "q"]), 40.0))
    X = t(G[pre + "X"])
    a = nk.ilu0_apply(fac, X, fused=True)
    b = nk.ilu0_apply(fac, X, fused=False)
    assert torch.equal(a, b)


def test_ilu0_singular_pivot_raises_like_reference(cuda):
    # newton_krylov.py:340-343: a singular pivot block raises RuntimeError
    # naming the element
    mk, kw, p = SPARSE_CASES["box3p_ns1"]
    d = Discretization(mk(), p, EquationSpec(**kw))
    A = nk.assemble_sparse_blocks(d, t(G["sp/box3p_ns1/q"]), 40.0)
    A.blocksT[A.entry(0, 0)].zero_()
    with pytest.raises(RuntimeError, match="singular ILU0 pivot block at element 0"):
        nk.ilu0_factor(A)


def test_sparse_blocks_and_ilu0_advection_diffusion_match_oracle(cuda):
    # scalar kind (one variable, viscous): not in the reference goldens, so
    # against the oracle restatement
    from oracle import solver_oracle as so
    from oracle.fr_oracle import OracleDisc
    m = mm.generate_box(3, 3, 2.0, 1.5)
    eqn = EquationSpec(kind="advection-diffusion", advection=(0.7, 0.4), diffusivity=0.02)
    d, o = Discretization(m, 2, eqn), OracleDisc(m, 2, eqn)
    q = np.random.default_rng(4).standard_normal(o.n_dofs)
    A = nk.assemble_sparse_blocks(d, t(q), 25.0)
    S = so.assemble_sparse(o, q, 25.0)
    assert np.array_equal(A.indices, S.indices)
    assert scaled(A.blocks, np.stack(S.blocks)) <= 1e-7
    X = np.random.default_rng(5).standard_normal(o.n_dofs)
    assert scaled(nk.ilu0_apply(nk.ilu0_factor(A), t(X)), so.ilu0_factor(S).apply(X)) <= 1e-6
