"""Device R / Jv at the BASELINE.json full sizes against the oracle, point
by point (VERDICT r1 "pin parity at the bench's full-size configs").

At these sizes two correct float64 evaluations that order their operations
differently disagree by far more than 1e-12: the reference itself and the
oracle differ by 1.2e-9 (max-norm, relative) at config 2 and by 1.3e-7 at
the low-Mach config 3, where p = 1/(gamma Ma^2) = 7e5 dwarfs R.  So each
float64 R is measured against one extended-precision truth -- the oracle's
algorithm in x87 long double on the same float64 operators, geometry and
input (``OracleDisc(..., dtype=np.longdouble).residual_mt``) -- and the
device must be at least as close to it as the reference's own float64
arithmetic, whose distance ``tests/golden/make_fullsize_floors.py`` measured
by running the reference (``fullsize_floors.json``):

* R at configs 2 (6.55 M DoF, the bench workload), 3, 4 (walls, stretched
  channel) and 5 (151 M DoF): device-vs-truth <= max(reference-vs-truth,
  1e-12) (reference spatial.py:501-570); the device-vs-oracle distance is
  printed next to it.
* Jv = s X - (R(q + eps X) - R0) / eps at config 2 with X of O(1) entries
  (the scaling of the reference golden ``c1/v``) against the truth's FD
  product of the same float64 q + eps X: <= 1e-9 (the reference's own
  float64 Jv is 3.5e-10 from it).
* the device R and Jv of the reference's own config-1 field against the
  vectors the *reference* produced (``G["c1/R0"]``, ``G["c1/Jv"]``)
  directly, not only through the oracle: <= 1e-12 and <= 1e-9.
* one ESDIRK3 JFNK-pMG step with the bench's config-2 settings (p{4-2},
  GMRES(30), rtol 1e-3, smoother_shift 5000, ptc.dtau_init = dt) on a
  48 x 48 version of config 2, against the REFERENCE's own step
  (golden_c2step.npz): PTC counts exact, every linear solve's GMRES count
  +-1 (restarted GMRES(30) solves of 73-148 iterations), solution <= 1e-7.
* config 3 at 128 x 128: the first three pmg_solve iterations against the
  reference's own run (golden_c3.npz).
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import _lib, cases
from paper_2202_09733_b200 import time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.spatial import Discretization

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).parent / "golden" / "golden.npz")
FLOORS = json.loads((Path(__file__).parent / "golden" / "fullsize_floors.json").read_text())


def _rel(dev, ref):
    d = dev.cpu().numpy() if isinstance(dev, torch.Tensor) else np.asarray(dev)
    return float(np.max(np.abs(d - ref)) / np.max(np.abs(ref)))


def _host_memory_gb():
    import psutil
    return psutil.virtual_memory().available / 2 ** 30


def _rel_ld(dev, truth):
    d = dev.cpu().numpy() if isinstance(dev, torch.Tensor) else np.asarray(dev)
    return float(np.max(np.abs(d.astype(np.longdouble) - truth)) / np.max(np.abs(truth)))


def _case(k, variant=None):
    """BASELINE config k; config 4's "adiabatic" variant swaps the isothermal
    no-slip wall (not in the reference) for the reference's adiabatic one on
    the same stretched channel -- the case the reference floor was measured
    on (tests/golden/make_fullsize_floors.py)."""
    import dataclasses

    from paper_2202_09733_b200 import mesh as mm
    c = cases.config(k)
    if variant == "adiabatic":
        yn = np.unique(c.mesh.nodes[:, 1])
        c = dataclasses.replace(c, mesh=mm.generate_channel(512, 128, 4.0, yn, bottom="wall-adiabatic"),
                                eqn=dataclasses.replace(c.eqn, wall_temperature=None))
    return c


@pytest.mark.parametrize("k,variant", [(2, None), (3, None), (4, "adiabatic"), (4, None), (5, None)])
def test_fullsize_residual_matches_oracle(cuda, k, variant):
    if k == 5 and _host_memory_gb() < 64:
        pytest.fail(f"config 5 oracle needs ~40 GB of host memory, {_host_memory_gb():.0f} GB available")
    c = _case(k, variant)
    d = Discretization(c.mesh, c.p, c.eqn)
    path = d.residual_path()
    R = d.residual(torch.as_tensor(c.q0, device="cuda")).cpu().numpy()
    del d
    torch.cuda.empty_cache()
    truth = OracleDisc(c.mesh, c.p, c.eqn, dtype=np.longdouble).residual_mt(c.q0)
    err = _rel_ld(R, truth)
    floor = FLOORS[f"config{k}"]["reference_R_vs_truth"]
    # the isothermal wall has no reference counterpart: its bound is twice
    # the reference's floor on the same geometry with the adiabatic wall
    tol = max(floor, 1e-12) * (2.0 if (k == 4 and variant is None) else 1.0)
    msg = f"config {k}{' ' + variant if variant else ''} ({path} kernels): {c.n_dofs} DoF, R vs long-double " \
          f"truth {err:.3e} (reference {floor:.3e})"
    if k != 5:
        msg += f", vs float64 oracle {_rel(R, OracleDisc(c.mesh, c.p, c.eqn).residual_mt(c.q0)):.3e}"
    print(msg)
    assert err <= tol


def test_fullsize_jv_matches_oracle(cuda):
    c = cases.config(2)
    jv = FLOORS["config2"]["jv"]
    d = Discretization(c.mesh, c.p, c.eqn)
    X = np.random.default_rng(jv["seed"]).uniform(-1.0, 1.0, c.n_dofs)
    shift, eps = jv["shift"], jv["eps"]
    q = torch.as_tensor(c.q0, device="cuda")
    R0 = d.residual(q)
    out = torch.empty_like(q)
    d.eval(q, _lib.EPI_JV, out, X=torch.as_tensor(X, device="cuda"), eps=eps, s=shift, R0=R0)
    tl = OracleDisc(c.mesh, c.p, c.eqn, dtype=np.longdouble)
    qp = c.q0 + eps * X  # float64, the reference's rounding (newton_krylov.py:76)
    Jt = shift * X.astype(np.longdouble) - (tl.residual_mt(qp) - tl.residual_mt(c.q0)) / eps
    err = _rel_ld(out, Jt)
    print(f"config 2 Jv vs long-double truth {err:.3e} (reference {FLOORS['config2']['reference_Jv_vs_truth']:.3e})")
    assert err <= 1e-9


def test_config1_residual_matches_reference_golden_directly(cuda):
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    assert np.array_equal(c.q0, G["c1/q0"])
    q = torch.as_tensor(G["c1/q0"], device="cuda")
    R0 = d.residual(q)
    assert _rel(R0, G["c1/R0"]) <= 1e-12
    # Jv against the reference's own FD product (newton_krylov.py:71-76);
    # measured floor 1.4e-10
    from paper_2202_09733_b200 import newton_krylov as nk
    Jv = nk.jfnk_matvec(torch.as_tensor(G["c1/v"], device="cuda"), q, R0, d.residual, 3.7)
    assert _rel(Jv, G["c1/Jv"]) <= 1e-9


def test_esdirk3_step_bench_config2_settings_matches_reference(cuda):
    """One ESDIRK3 JFNK-pMG step with the bench's config-2 settings on a
    48 x 48 version of config 2, against the REFERENCE's own step
    (tests/golden/make_golden_c2step.py: its esdirk_step + ImplicitDriver
    with the derived ESDIRK3 tableau injected; 1097 s on one core).  These
    are restarted GMRES(30) solves of 73-148 iterations each (the oracle
    restatement itself lands within +-1 of every one)."""
    GS = np.load(Path(__file__).parent / "golden" / "golden_c2step.npz")
    c = cases.config(2, nx=48)
    import hashlib
    assert hashlib.sha256(c.q0.tobytes()).hexdigest() == str(GS["q0_sha256"]) and float(GS["dt"]) == c.dt
    d = Discretization(c.mesh, c.p, c.eqn)
    s = ti.get_scheme("esdirk3")
    cfg = {"case.precond": "pmg", "pmg.levels": c.levels, "pmg.smooth": "2",
           "pmg.smoother_shift": c.extra["smoother_shift"], "gmres.kdim": 30, "gmres.rtol": 1e-3,
           "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4}
    q_d, info = ImplicitDriver(d, cfg).step(torch.as_tensor(c.q0, device="cuda"), c.dt, s)
    ptc_d = [i["iters"] for i in info]
    gm_d = [x for i in info for x in i["gmres_per_iter"]]
    gm_r = list(GS["gmres_counts"])
    err = _rel(q_d, GS["q1"])
    print(f"48^2 config-2 settings: PTC {ptc_d} vs {list(GS['ptc_iters'])}, GMRES per solve {gm_d} vs {gm_r}, "
          f"solution {err:.3e}")
    assert ptc_d == list(GS["ptc_iters"])
    assert len(gm_d) == len(gm_r) and all(abs(x - y) <= 1 for x, y in zip(gm_d, gm_r))
    assert err <= 1e-7


def test_config3_pmg_solve_history_matches_reference_full_size(cuda):
    """BASELINE config 3 at its full 128 x 128 size: the first three outer
    iterations of the nonlinear pMG solver (pmg.py:308-374) over
    p{4-3-2-1-0} with EJ on every level, against the REFERENCE's own run
    (tests/golden/make_golden_c3.py, golden_c3.npz).  At Ma = 1e-3 the
    pressure (7e5) dwarfs R, whose float64 evaluations differ by 1.3e-7 of
    its max between the reference and the oracle (fullsize_floors.json).
    The oracle's own run (OracleDisc + solver_oracle.pmg_solve, 172 s on 8
    cores) differs from the reference's by 9e-6 in the history and, per
    conserved variable (max error / max magnitude over the sampled state),
    by ORACLE_FLOOR below -- 2.2e-3 in y-momentum, whose magnitude (5e-5)
    is the 1e-6 seeded noise.  The device must agree with the reference to
    1e-4 in the history and to twice the oracle's floor per variable."""
    from paper_2202_09733_b200 import newton_krylov as nk, pmg
    GC = np.load(Path(__file__).parent / "golden" / "golden_c3.npz")
    c = cases.config(3)
    d = Discretization(c.mesh, c.p, c.eqn)
    h = pmg.PHierarchy.parse(c.levels, "2", "ej")
    ctx = pmg.PmgContext(d, pmg.PmgPrecondConfig(h, smoother_shift=c.extra["smoother_shift"]))
    q, st = pmg.pmg_solve(ctx, torch.as_tensor(c.q0, device="cuda"),
                          nk.PtcConfig(dtau_init=0.1, max_iters=int(GC["iters"]), rtol=1e-14))
    hist = np.array(st["history"])
    ref = GC["history"]
    Q = q.cpu().numpy().reshape(c.mesh.n_elements, -1)
    S = Q[::int(GC["sub_stride"])].reshape(-1, 4)
    Sr = GC["q_sub"].reshape(-1, 4)
    per_var = np.max(np.abs(S - Sr), axis=0) / np.max(np.abs(Sr), axis=0)
    sums = Q.reshape(len(Q), -1, 4).sum(axis=(0, 1))
    print("config 3 history device", hist[:, 1].tolist(), "reference", ref[:, 1].tolist(),
          "state per variable", per_var.tolist(), "sums", sums.tolist(), GC["q_sum"].tolist())
    assert hist.shape == ref.shape
    assert np.allclose(hist[:, 1], ref[:, 1], rtol=1e-4, atol=0.0)
    assert np.allclose(hist[:, 2], ref[:, 2], rtol=1e-4, atol=0.0)   # the SER pseudo-time steps
    ORACLE_FLOOR = np.array([8.6e-12, 8.2e-8, 2.23e-3, 5.3e-12])   # oracle vs reference, measured
    assert np.all(per_var <= np.maximum(2.0 * ORACLE_FLOOR, 1e-10))
