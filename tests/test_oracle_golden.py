"""Pin the oracle (CPU restatement) to the reference's own outputs.

Fixtures: tests/golden/golden.npz, produced by running the reference
pmgflow in the build container (tests/golden/make_golden.py)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import solver_oracle as so
from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import cases, mesh as mm, operators as ops
from paper_2202_09733_b200.equation import EquationSpec
from paper_2202_09733_b200.time_integration import get_scheme

G = np.load(Path(__file__).parent / "golden" / "golden.npz")

MESHES = {
    "box4p": lambda: mm.generate_box(4, 4, 1.0, 1.0, periodic=True),
    "box3ff": lambda: mm.generate_box(3, 3, 2.0, 1.5),
    "cyl_adiab": lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3),
    "cyl_slip": lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3, wall_tag="wall-slip"),
}
KINDS = {
    "euler": dict(kind="euler", mach=0.3),
    "ns": dict(kind="navier-stokes", mach=0.3, reynolds=200.0),
    "advd": dict(kind="advection-diffusion", advection=(0.7, 0.4), diffusivity=0.02),
}


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_operators_match_reference():
    for p in range(6):
        b = ops.basis(p)
        assert np.allclose(b.diff_matrix, G[f"ops/p{p}/D"], rtol=0, atol=1e-12)
        assert np.allclose(b.weights, G[f"ops/p{p}/w"], rtol=0, atol=1e-15)
    for pf in range(1, 6):
        for pc in range(pf):
            t = ops.transfer_operators(pf, pc)
            assert np.allclose(t.gamma, G[f"ops/T{pf}{pc}/gamma"], atol=1e-13)
            assert np.allclose(t.pi, G[f"ops/T{pf}{pc}/pi"], atol=1e-13)


@pytest.mark.parametrize("name", ["box4p", "box3ff", "cyl"])
def test_mesh_matches_reference(name):
    m = {"box4p": MESHES["box4p"], "box3ff": MESHES["box3ff"], "cyl": MESHES["cyl_adiab"]}[name]()
    assert np.array_equal(m.interior_faces, G[f"mesh/{name}/interior_faces"])
    assert np.array_equal(m.boundary_faces, G[f"mesh/{name}/boundary_faces"])
    g = mm.element_geometry(m, 3)
    assert np.allclose(g.det, G[f"mesh/{name}/det"], rtol=1e-14, atol=0)
    assert np.allclose(g.face_normals, G[f"mesh/{name}/normals"], atol=1e-15)
    assert np.allclose(g.face_jac, G[f"mesh/{name}/face_jac"], rtol=1e-15)


@pytest.mark.parametrize("mesh", list(MESHES))
@pytest.mark.parametrize("kind", list(KINDS))
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_oracle_residual_matches_reference(mesh, kind, p):
    d = OracleDisc(MESHES[mesh](), p, EquationSpec(**KINDS[kind]))
    q = G[f"res/{mesh}/{kind}/p{p}/q"]
    assert rel(d.residual(q), G[f"res/{mesh}/{kind}/p{p}/R"]) <= 1e-13


def test_oracle_blocks_match_reference():
    m = mm.generate_box(3, 3, 1.0, 1.0, periodic=True)
    d = OracleDisc(m, 2, EquationSpec(kind="navier-stokes", mach=0.3, reynolds=100.0))
    q = G["blk/q"]
    B = so.assemble_blocks(d, q, 30.0)
    scale = np.abs(G["blk/blocks"]).max()
    assert np.abs(B.blocks - G["blk/blocks"]).max() / scale <= 1e-7
    assert rel(B.apply(G["blk/X"]), G["blk/Y"]) <= 1e-7
    fr = d.freeze(q)
    Q = q[d.offsets[4]:d.offsets[5]].reshape(3, 3, 4) * 1.001
    assert rel(d.element_residual(4, Q, fr), G["blk/local_e4"]) <= 1e-13


def test_oracle_config1_residual_and_jv():
    c = cases.config(1)
    assert np.array_equal(c.q0, G["c1/q0"])
    d = OracleDisc(c.mesh, c.p, c.eqn)
    R0 = d.residual(c.q0)
    assert rel(R0, G["c1/R0"]) <= 1e-12  # north-star tolerance; floor 1.5e-13 (A.5)
    Jv = so.jfnk_matvec(G["c1/v"], c.q0, R0, d.residual, 3.7)
    # FD epsilon amplifies rounding by 1/eps: floor 1.4e-10
    assert rel(Jv, G["c1/Jv"]) <= 1e-8
    v = G["c1/v"]
    Jvu = so.jfnk_matvec(v / np.linalg.norm(v), c.q0, R0, d.residual, 3.7)
    assert rel(Jvu, G["c1/Jvu"]) <= 1e-6


def test_oracle_precondition_matches_reference():
    c = cases.config(1)
    d = OracleDisc(c.mesh, c.p, c.eqn)
    ctx = so.Pmg(d, "3-2", 2, smoother_shift=50.0)
    ctx.prepare(c.q0, float(G["c1/pc_shift"]))
    v = G["c1/v"]
    Y = ctx.precondition(v / np.linalg.norm(v))
    assert rel(Y, G["c1/pc_Y"]) <= 1e-8


def test_oracle_esdirk2_step_matches_reference():
    c = cases.config(1)
    d = OracleDisc(c.mesh, c.p, c.eqn)
    drv = so.Driver(d, "pmg", "3-2", 2, smoother_shift=50.0, gmres_rtol=1e-3, dtau_init=c.dt)
    s = get_scheme("esdirk2")
    q1 = drv.esdirk_step(c.q0, c.dt, s.a, s.b)
    counts = [n for rec in drv.records for n in rec[3]]
    ref = list(G["c1/esdirk2/gmres_counts"])
    assert len(counts) == len(ref)
    assert all(abs(a - b) <= 1 for a, b in zip(counts, ref))
    assert [rec[1] for rec in drv.records] == list(G["c1/esdirk2/ptc_iters"])
    # solution floor 1.2e-8
    assert rel(q1, G["c1/esdirk2/q1"]) <= 1e-7


def test_oracle_row4_step_matches_reference():
    c = cases.config(1)
    d = OracleDisc(c.mesh, c.p, c.eqn)
    drv = so.Driver(d, "pmg", "3-2", 2, smoother_shift=50.0, gmres_rtol=1e-3)
    s = get_scheme("row4")
    q1 = drv.row_step(c.q0, c.dt, s.a, s.cmat, s.b, s.gamma)
    counts = [rec[2] for rec in drv.records]
    ref = list(G["c1/row4/gmres_counts"])
    assert all(abs(a - b) <= 1 for a, b in zip(counts, ref)) and len(counts) == len(ref)
    assert rel(q1, G["c1/row4/q1"]) <= 1e-6


def test_oracle_pmg_solve_matches_reference():
    c = cases.config(3, nx=4)
    assert np.array_equal(c.q0, G["c3/q0"])
    d = OracleDisc(c.mesh, 4, c.eqn)
    ctx = so.Pmg(d, "4-3-2-1-0", 2, smoother_shift=1e3)
    q, st = so.pmg_solve(ctx, c.q0, 0.1, max_iters=6, rtol=1e-10)
    h = np.array(st["history"])
    ref = G["c3/history"]
    assert h.shape == ref.shape
    # Ma = 1e-3: E ~ 1.8e6, so the absolute FD eps is ~5e-13 of the state and
    # the FD blocks amplify rounding; histories agree to ~1e-3
    assert np.allclose(h[:, 1], ref[:, 1], rtol=2e-3, atol=1e-12)
    assert rel(q, G["c3/q"]) <= 1e-9


@pytest.mark.parametrize("mesh", list(MESHES))
@pytest.mark.parametrize("kind", list(KINDS))
def test_oracle_threaded_residual_is_bitwise_identical(mesh, kind):
    # bench.py's reference arm runs residual_mt on all host cores: it must be
    # the same computation as residual, chunking included
    d = OracleDisc(MESHES[mesh](), 3, EquationSpec(**KINDS[kind]))
    q = G[f"res/{mesh}/{kind}/p3/q"]
    assert np.array_equal(d.residual_mt(q, threads=3, chunk=5), d.residual(q))


def test_oracle_threaded_residual_raises_like_residual():
    from paper_2202_09733_b200.equation import NonPhysicalStateError
    d = OracleDisc(MESHES["box4p"](), 2, EquationSpec(**KINDS["ns"]))
    q = G["res/box4p/ns/p2/q"].copy().reshape(16, 3, 3, 4)
    q[11, 1, 1, 0] = -1.0   # negative density at an interior point of element 11
    q[6, 0, 0, 3] = 0.0     # negative pressure at a corner point of element 6
    errs = []
    for f in (d.residual, lambda x: d.residual_mt(x, threads=4, chunk=3)):
        with pytest.raises(NonPhysicalStateError) as ei:
            f(q.reshape(-1))
        errs.append(str(ei.value))
    assert errs[0] == errs[1]


def test_oracle_long_double_truth_pins_reference_config1():
    # the extended-precision oracle the full-size parity tests use as truth
    # (tests/test_gpu_fullsize_oracle.py) agrees with the reference's own
    # float64 config-1 residual to the reference's rounding floor
    c = cases.config(1)
    tl = OracleDisc(c.mesh, c.p, c.eqn, dtype=np.longdouble)
    truth = tl.residual(c.q0)
    assert truth.dtype == np.longdouble
    assert np.array_equal(truth, tl.residual_mt(c.q0))
    err = float(np.max(np.abs(G["c1/R0"] - truth)) / np.max(np.abs(truth)))
    assert err <= 1e-12
