"""Oracle MBNK path (block-sparse FD Jacobian, block ILU0, MBNK smoother,
switch_after) against goldens made by running the reference
(tests/golden/make_golden_mbnk.py).  FD blocks carry the reference's own
FD noise (R rounding x 1/eps, eps = 1e-6), hence ~1e-7-of-scale tolerances."""

from pathlib import Path

import numpy as np
import pytest

from oracle import solver_oracle as so
from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import cases, mesh as mm
from paper_2202_09733_b200.equation import EquationSpec

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
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name", list(SPARSE_CASES))
def test_oracle_sparse_blocks_and_ilu0_match_reference(name):
    mk, kw, p = SPARSE_CASES[name]
    d = OracleDisc(mk(), p, EquationSpec(**kw))
    pre = f"sp/{name}/"
    q, X = G[pre + "q"], G[pre + "X"]
    S = so.assemble_sparse(d, q, 40.0)
    assert np.array_equal(S.indptr, G[pre + "indptr"]) and np.array_equal(S.indices, G[pre + "indices"])
    assert scaled(np.stack(S.blocks), G[pre + "blocks"]) <= 1e-7
    fac = so.ilu0_factor(S)
    assert scaled(np.stack(fac.F.blocks), G[pre + "lu"]) <= 1e-6
    assert scaled(np.stack(fac.diag_inv), G[pre + "dinv"]) <= 1e-6
    assert scaled(S.matvec(X), G[pre + "AX"]) <= 1e-7
    assert scaled(fac.apply(X), G[pre + "iluX"]) <= 1e-6


@pytest.mark.parametrize("kinds", ["mbnk", "ej-mbnk"])
def test_oracle_mbnk_precondition_matches_reference(kinds):
    c = cases.config(1, nx=4)
    d = OracleDisc(c.mesh, 3, c.eqn)
    ctx = so.Pmg(d, "3-2", 1, smoother_shift=50.0, smoother=kinds)
    ctx.prepare(G["mb/q"], float(G["mb/shift"]))
    assert scaled(ctx.precondition(G["mb/v"]), G[f"mb/{kinds}/Y"]) <= 1e-6


def test_oracle_switch_after_matches_reference():
    c = cases.config(1, nx=4)
    d = OracleDisc(c.mesh, 3, c.eqn)
    ctx = so.Pmg(d, "3-2", 1, smoother_shift=50.0, switch_after=1)
    q, st = so.pmg_solve(ctx, G["sw/q0"], 0.05, max_iters=3, rtol=1e-12)
    h, ref = np.array(st["history"]), G["sw/history"]
    assert h.shape == ref.shape
    assert np.allclose(h[:, 1], ref[:, 1], rtol=1e-5)
    assert scaled(q, G["sw/q"]) <= 1e-7
