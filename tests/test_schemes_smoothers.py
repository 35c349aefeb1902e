"""CPU checks of the two BASELINE items the reference does not ship
(SURVEY 8.0): the derived ESDIRK3 tableau and the pseudo-transient RK
smoother (north star item 3).

ESDIRK3 is pinned to the reference: its tableau was injected into the
reference's own esdirk_step / ImplicitDriver and validate_tableau
(tests/golden/make_golden_esdirk3.py).  The RK smoother has no reference
counterpart: its oracle restatement (solver_oracle.rk_spectral_radius,
Pmg._smooth "rk") is checked here by construction and by property
("parity unpinned" vs the reference).
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import solver_oracle as so
from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import cases, mesh as mm, pmg
from paper_2202_09733_b200 import time_integration as ti
from paper_2202_09733_b200.equation import EquationSpec
from paper_2202_09733_b200.harness import DEFAULTS, pmg_precond_config
from paper_2202_09733_b200.operators import fr_advection_radius, rk_adv_coef

GE = np.load(Path(__file__).parent / "golden" / "golden_esdirk3.npz")


def test_esdirk3_tableau_is_the_one_the_reference_validated():
    s = ti.get_scheme("esdirk3")
    assert np.array_equal(s.a, GE["tableau/a"])
    assert GE["tableau/checks"].all(), dict(zip(GE["tableau/check_names"], GE["tableau/checks"]))
    g = s.a[1, 1]
    assert abs(g ** 3 - 3 * g * g + 1.5 * g - 1.0 / 6.0) < 1e-15
    c = s.a.sum(axis=1)
    b = s.b
    assert np.array_equal(b, s.a[-1])                    # stiffly accurate
    assert abs(b.sum() - 1.0) < 1e-15
    assert abs(b @ c - 0.5) < 1e-15
    assert abs(b @ c ** 2 - 1.0 / 3.0) < 1e-15
    assert abs(b @ (s.a @ c) - 1.0 / 6.0) < 1e-15
    # L-stability: R(-1e6) -> 0 (reference stability_function)
    R = GE["tableau/R"]
    assert abs(R[0]) < 1e-5
    assert np.all(np.abs(R[3:6]) <= 1.0 + 1e-12)


@pytest.mark.slow
def test_oracle_esdirk3_step_matches_reference():
    c = cases.config(1)
    o = OracleDisc(c.mesh, c.p, c.eqn)
    s = ti.get_scheme("esdirk3")
    drv = so.Driver(o, "pmg", "3-2", 2, smoother_shift=50.0, gmres_rtol=1e-3, dtau_init=c.dt)
    q1 = drv.esdirk_step(c.q0, c.dt, s.a, s.b)
    counts = [n for r in drv.records for n in r[3]]
    ref = list(GE["c1/esdirk3/gmres_counts"])
    assert len(counts) == len(ref) and all(abs(a - b) <= 1 for a, b in zip(counts, ref)), (counts, ref)
    assert [r[1] for r in drv.records] == list(GE["c1/esdirk3/ptc_iters"])
    assert np.max(np.abs(q1 - GE["c1/esdirk3/q1"])) / np.max(np.abs(GE["c1/esdirk3/q1"])) <= 1e-7


def test_rk_spectral_radius_free_stream():
    # uniform free stream on a uniform box: lambda = A_p (|u|+c)/h + (p+1)^4 nu/h^2
    m = mm.generate_box(4, 3, 2.0, 3.0, periodic=True)
    eqn = EquationSpec(kind="navier-stokes", mach=0.4, reynolds=50.0, ref_length=2.0)
    p = 3
    o = OracleDisc(m, p, eqn)
    q = np.tile(eqn.free_stream(), o.n_dofs // 4)
    lam = so.rk_spectral_radius(o, q)
    rho, u, v, E = eqn.free_stream()
    pr = (eqn.gamma - 1.0) * (E - 0.5 * (u * u + v * v) / rho)
    a = np.hypot(u / rho, v / rho) + np.sqrt(eqn.gamma * pr / rho)
    h = 0.5  # 0.5 x 1.0 cells: 4 |det| / max(L) = 4 (0.25 * 0.5) / 1.0
    nu = max(4.0 / 3.0 * eqn.mu, eqn.heat_conductivity * (eqn.gamma - 1.0)) / rho
    ref = rk_adv_coef(p) * a / h + (p + 1) ** 4 * nu / h ** 2
    assert np.allclose(lam, ref, rtol=1e-14, atol=0)
    # scalar advection-diffusion: state independent
    e2 = EquationSpec(kind="advection-diffusion", advection=(0.6, 0.8), diffusivity=0.01)
    o2 = OracleDisc(m, 2, e2)
    lam2 = so.rk_spectral_radius(o2, np.zeros(o2.n_dofs))
    assert np.allclose(lam2, rk_adv_coef(2) * 1.0 / h + 81 * 0.01 / h ** 2, rtol=1e-14)


def test_fr_advection_radius():
    # p = 0 is first-order upwind FV (radius 2/h = 2 rho_0 / h), p = 1 is 3;
    # larger p grow faster than 2p+1 (Bloch analysis of the FR operator)
    assert abs(fr_advection_radius(0) - 1.0) < 1e-13
    assert abs(fr_advection_radius(1) - 3.0) < 1e-12
    r = [fr_advection_radius(p) for p in range(6)]
    assert all(b > a for a, b in zip(r, r[1:]))
    assert 13.8 < r[4] < 14.0 and 18.8 < r[5] < 19.0
    assert rk_adv_coef(3) == 2.0 * np.sqrt(2.0) * r[3]


def test_rk_smoother_contracts_the_level_defect():
    # twenty sweeps on a single level reduce ||defect|| (after a non-normal
    # transient growth of the first sweeps; measured ratios after 1 / 10 /
    # 20 / 40 sweeps: 1.18, 0.86, 0.38, 0.10)
    c = cases.config(1, nx=6)
    o = OracleDisc(c.mesh, c.p, c.eqn)
    ctx = so.Pmg(o, "3", 20, smoother="rk")
    shift = 1.0 / (0.43 * c.dt) + 1.0 / c.dt
    ctx.prepare(c.q0, shift)
    lev = ctx.levels[0]
    assert lev.blocks is None and lev.lam.shape == (o.mesh.n_elements,) and np.all(lev.lam > 0)
    rng = np.random.default_rng(3)
    X = rng.standard_normal(o.n_dofs)
    lev.q = c.q0.copy()
    lev.S_base = shift * c.q0 - o.residual(c.q0)
    lev.S_extra = 1e-3 * X / np.linalg.norm(X)
    d0 = np.linalg.norm(lev.defect())
    ctx._smooth(0)
    d1 = np.linalg.norm(lev.defect())
    assert d1 < 0.5 * d0, (d0, d1)


@pytest.mark.slow
def test_oracle_rk_ej_preconditioned_step_converges():
    c = cases.config(1, nx=8)
    o = OracleDisc(c.mesh, c.p, c.eqn)
    s = ti.get_scheme("esdirk2")
    drv = so.Driver(o, "pmg", "3-2", 2, smoother_shift=50.0, gmres_rtol=1e-3, dtau_init=c.dt, smoother="rk-ej")
    drv.esdirk_step(c.q0, c.dt, s.a, s.b)
    assert all(r[1] <= 6 for r in drv.records)
    assert all(r[2] <= 80 for r in drv.records)


def test_rk_hierarchy_parse_and_config():
    h = pmg.PHierarchy.parse("5-4", "2", "rk-ej")
    assert h.smoothers == ("rk", "ej")
    with pytest.raises(ValueError):
        pmg.PHierarchy.parse("3-2", "2", "rk-gs")
    cfg = dict(DEFAULTS)
    cfg.update({"pmg.levels": "3-2-1", "pmg.smoother": "rk-rk-ej", "pmg.rk.cfl": 1.2,
                "pmg.rk.stages": "0.5,1.0"})
    pc = pmg_precond_config(cfg)
    assert pc.rk_cfl == 1.2 and pc.rk_alphas == (0.5, 1.0)
    assert pc.hierarchy.smoothers == ("rk", "rk", "ej")
    with pytest.raises(ValueError):
        pmg.PmgPrecondConfig(h, rk_cfl=0.0)


# ---------------------------------------------------------------------------
# Rusanov / LDG options of the oracle (BASELINE interface schemes)

@pytest.mark.parametrize("riemann,visc", [("rusanov", "br1"), ("roe", "ldg"), ("rusanov", "ldg")])
def test_oracle_options_conservative_and_free_stream(riemann, visc):
    m = mm.generate_box(4, 4, 2.0, 2.0, periodic=True)
    eqn = EquationSpec(kind="navier-stokes", mach=0.3, reynolds=100.0, riemann=riemann, viscous_scheme=visc)
    o = OracleDisc(m, 3, eqn)
    qf = o.free_stream_field()
    assert np.max(np.abs(o.residual(qf))) <= 1e-11
    rng = np.random.default_rng(2)
    q = qf * (1.0 + 0.01 * rng.standard_normal(qf.shape))
    R = o.residual(q).reshape(-1, 4, 4, 4)
    from paper_2202_09733_b200.operators import gauss_rule
    w = gauss_rule(4)[1]
    tot = np.einsum("a,b,mab,mabv->v", w, w, o.det, R)
    assert np.max(np.abs(tot)) <= 1e-11 * np.max(np.abs(R))


def test_rusanov_consistency_and_dissipation():
    from oracle.fr_oracle import euler_flux, roe_flux, rusanov_flux
    rng = np.random.default_rng(4)
    g = 1.4
    q = np.stack([1 + 0.1 * rng.random(50), rng.random(50), rng.random(50), 3 + rng.random(50)], axis=-1)
    th = rng.random(50) * 2 * np.pi
    nrm = np.stack([np.cos(th), np.sin(th)], axis=-1)
    fx, fy = euler_flux(q, g)
    exact = fx * nrm[:, :1] + fy * nrm[:, 1:]
    assert np.allclose(rusanov_flux(q, q, nrm, g), exact, rtol=1e-14, atol=1e-14)
    # Rusanov dissipates at least as much as Roe on a density jump
    q2 = q.copy()
    q2[:, 0] *= 1.2
    d_rus = np.abs(rusanov_flux(q, q2, nrm, g) - 0.5 * (exact + (euler_flux(q2, g)[0] * nrm[:, :1]
                                                               + euler_flux(q2, g)[1] * nrm[:, 1:])))
    d_roe = np.abs(roe_flux(q, q2, nrm, g) - 0.5 * (exact + (euler_flux(q2, g)[0] * nrm[:, :1]
                                                             + euler_flux(q2, g)[1] * nrm[:, 1:])))
    assert np.all(d_rus[:, 0] >= d_roe[:, 0] - 1e-12)
    with pytest.raises(ValueError):
        EquationSpec(kind="euler", riemann="hllc")
    with pytest.raises(ValueError):
        EquationSpec(kind="euler", viscous_scheme="ip")


GR = np.load(Path(__file__).parent / "golden" / "golden_ros4l.npz")


def _ros4l_original_form():
    """Recover (A, B, b) of the original (alpha, beta = alpha + gamma)
    form from the K form: G = (diag(1/g) - C)^-1, A = a G, b = m G."""
    s = ti.get_scheme("ros4l")
    G = np.linalg.inv(np.eye(4) / s.gamma - s.cmat)
    A = s.a @ G
    b = s.b @ G
    B = A + G - s.gamma * np.eye(4)
    return s, A, B, b


def test_ros4l_order_conditions_and_reference_checks():
    s, A, B, b = _ros4l_original_form()
    g = s.gamma
    al, bp = A.sum(1), B.sum(1)
    conds = [b.sum() - 1, b @ bp - (0.5 - g), b @ al ** 2 - 1 / 3, b @ B @ bp - (1 / 6 - g + g * g),
             b @ al ** 3 - 0.25, (b * al) @ A @ bp - (1 / 8 - g / 3), b @ B @ al ** 2 - (1 / 12 - g / 3),
             b @ B @ B @ bp - (1 / 24 - g / 2 + 1.5 * g * g - g ** 3)]
    assert np.max(np.abs(conds)) < 1e-14, conds
    assert abs(g ** 4 - 4 * g ** 3 + 3 * g * g - 2 * g / 3 + 1 / 24) < 1e-15
    # the tableau the reference's validate_tableau passed (make_golden_ros4l.py)
    assert np.array_equal(s.a, GR["tableau/a"]) and np.array_equal(s.cmat, GR["tableau/cmat"])
    assert np.array_equal(s.b, GR["tableau/m"])
    assert GR["tableau/checks"].all(), dict(zip(GR["tableau/check_names"], GR["tableau/checks"]))
    R = GR["tableau/R"]
    assert abs(R[0]) < 1e-5                                   # L-stable
    assert np.all(np.abs(R[3:6]) <= 1.0 + 1e-12)              # |R(iy)| <= 1
    for z in GR["tableau/z"]:
        assert abs(ti.stability_function(s, z) - R[list(GR["tableau/z"]).index(z)]) < 1e-13


def test_ros4l_empirical_order_four():
    """The K-form stage algebra of row_step with an exact Jacobian on a
    nonlinear (van der Pol, mu = 1) system: error ratios -> 2^4."""
    from scipy.integrate import solve_ivp
    s = ti.get_scheme("ros4l")
    f = lambda y: np.array([y[1], (1 - y[0] ** 2) * y[1] - y[0]])
    J = lambda y: np.array([[0.0, 1.0], [-2 * y[0] * y[1] - 1.0, 1 - y[0] ** 2]])
    y0 = np.array([2.0, 0.0])
    ref = solve_ivp(lambda t, y: f(y), (0, 1.0), y0, rtol=1e-13, atol=1e-14, method="DOP853").y[:, -1]
    errs = []
    for N in (10, 20, 40, 80):
        y, h = y0.copy(), 1.0 / N
        for _ in range(N):
            W = np.eye(2) / (s.gamma * h) - J(y)
            K = []
            for i in range(4):
                yi = y + sum(s.a[i, j] * K[j] for j in range(i))
                K.append(np.linalg.solve(W, f(yi) + sum(s.cmat[i, j] / h * K[j] for j in range(i))))
            y = y + sum(s.b[j] * K[j] for j in range(4))
        errs.append(np.abs(y - ref).max())
    slopes = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(slopes > 3.8), (errs, slopes)


def test_oracle_ros4l_step_matches_reference():
    c = cases.config(1)
    o = OracleDisc(c.mesh, c.p, c.eqn)
    s = ti.get_scheme("ros4l")
    drv = so.Driver(o, "pmg", "3-2", 2, smoother_shift=50.0, gmres_rtol=1e-3)
    q1 = drv.row_step(c.q0, c.dt, s.a, s.cmat, s.b, s.gamma)
    counts = [rec[2] for rec in drv.records]
    ref = list(GR["c1/ros4l/gmres_counts"])
    assert len(counts) == len(ref) and all(abs(a - b) <= 1 for a, b in zip(counts, ref)), (counts, ref)
    assert np.max(np.abs(q1 - GR["c1/ros4l/q1"])) / np.max(np.abs(GR["c1/ros4l/q1"])) <= 1e-6


def test_oracle_gmres_cgs2_matches_mgs_kat():
    # gmres.ortho = cgs2 (classical Gram-Schmidt + one reorthogonalisation,
    # the partitioned solver's 3-all-reduce Arnoldi option): the same
    # Krylov iterates as the reference's MGS on a well-conditioned SPD
    # system, to rounding (reference tests/test_newton_krylov.py:29-48)
    from oracle import solver_oracle as so
    rng = np.random.default_rng(7)
    n = 40
    A = rng.standard_normal((n, n))
    A = A @ A.T + n * np.eye(n)
    b = rng.standard_normal(n)
    xm, im, rm = so.gmres_solve(lambda v: A @ v, b, kdim=5, max_restarts=60, rtol=1e-10)
    xc, ic, rc = so.gmres_solve(lambda v: A @ v, b, kdim=5, max_restarts=60, rtol=1e-10, ortho="cgs2")
    assert im == ic and rm <= 1e-10 and rc <= 1e-10
    assert np.allclose(xc, np.linalg.solve(A, b), atol=1e-8)
    assert np.max(np.abs(xc - xm)) <= 1e-12 * np.max(np.abs(xm))
