"""The drop-in, shown through the REFERENCE's own host code.

The reference package installed unmodified under baseline/_ref (the
reference arm's install) is imported as ``pmgflow``
and its own solvers are handed the device objects as their callables --
NumPy in, NumPy out, exactly the duck-typed seams of SURVEY 8(b):

* ``time_integration.esdirk_step`` + ``harness.ImplicitDriver``
  (time_integration.py:144-168, harness.py:277-369) with the device
  ``Discretization.residual`` as the ``residual`` callable: the PTC stage
  function evaluates R on the B200 while the reference drives PTC, GMRES
  and its own CPU pMG preconditioner.  Counts and state must match the
  reference's all-CPU step (golden_esdirk3.npz).
* ``newton_krylov.gmres_solve`` (newton_krylov.py:79-151) with the device
  fused Jv as ``matvec`` and the device element-Jacobi ``apply`` as
  ``precond``, against the same solve with the reference's CPU matvec and
  blocks.
* ``newton_krylov.ptc_solve`` (newton_krylov.py:377-437) with the device
  stage function as ``F`` and the device pMG ``prepare``/``precondition``
  as the preconditioner factory, against the re-hosted device PTC.

Skipped (not failed) when baseline/_ref is absent: it is git-ignored and
made by the reference-arm install command.
"""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
pytestmark = pytest.mark.gpu
if not (REF / "pmgflow").exists():
    pytest.skip("baseline/_ref (the reference install) is absent", allow_module_level=True)
sys.path.insert(0, str(REF))

from pmgflow import harness as rh  # noqa: E402
from pmgflow import mesh as rmesh  # noqa: E402
from pmgflow import newton_krylov as rnk  # noqa: E402
from pmgflow import spatial as rsp  # noqa: E402
from pmgflow import time_integration as rti  # noqa: E402

from paper_2202_09733_b200 import cases, newton_krylov as nk, pmg  # noqa: E402
from paper_2202_09733_b200 import time_integration as ti  # noqa: E402
from paper_2202_09733_b200.spatial import Discretization  # noqa: E402

G = np.load(ROOT / "tests" / "golden" / "golden_esdirk3.npz")
assert rsp.__file__.startswith(str(REF)), "must exercise the installed reference, not this repo"


def _rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def _ref_eqn(e):
    return rsp.EquationSpec(kind=e.kind, mach=e.mach, reynolds=e.reynolds, ref_length=e.ref_length,
                            gamma=e.gamma, prandtl=e.prandtl)


def _ref_scheme():
    s = ti.get_scheme("esdirk3")
    return rti.StageScheme(s.name, s.kind, s.order, s.a.copy(), s.b.copy(), s.c.copy())


class GmresCount:
    def __enter__(self):
        self.counts = []
        self._orig = rnk.gmres_solve

        def wrapped(*a, **k):
            x, it, rr = self._orig(*a, **k)
            self.counts.append(it)
            return x, it, rr
        rnk.gmres_solve = wrapped
        return self

    def __exit__(self, *exc):
        rnk.gmres_solve = self._orig


def test_reference_esdirk_step_drives_device_residual(cuda):
    c = cases.config(1)
    dev = Discretization(c.mesh, c.p, c.eqn)
    ref = rsp.Discretization(rmesh.generate_box(16, 16, 10.0, 10.0, periodic=True), 3, _ref_eqn(c.eqn))
    cfg = rh.parse_config_text(f"""
case.precond = pmg
pmg.levels = 3-2
pmg.smooth = 2
pmg.smoother_shift = 50
gmres.kdim = 30
gmres.rtol = 1e-3
ptc.dtau_init = {c.dt!r}
ptc.rtol = 1e-4
""")
    drv = rh.ImplicitDriver(ref, cfg)
    calls = []

    def residual(q):                      # the seam: NumPy in, NumPy out, R on the B200
        calls.append(1)
        return dev.residual(q)
    with GmresCount() as log:
        q1, info = rti.esdirk_step(c.q0, c.dt, _ref_scheme(), residual, drv.solve_stage)
    assert len(calls) > 50
    assert [i["iters"] for i in info] == list(G["c1/esdirk3/ptc_iters"])
    assert all(abs(a - b) <= 1 for a, b in zip(log.counts, G["c1/esdirk3/gmres_counts"])), log.counts
    assert _rel(q1, G["c1/esdirk3/q1"]) <= 1e-7


def test_reference_gmres_with_device_jv_and_ej(cuda):
    c = cases.config(1)
    dev = Discretization(c.mesh, c.p, c.eqn)
    ref = rsp.Discretization(rmesh.generate_box(16, 16, 10.0, 10.0, periodic=True), 3, _ref_eqn(c.eqn))
    q = c.q0
    shift = 40.0
    b = np.random.default_rng(3).standard_normal(q.size)
    kc = rnk.KrylovConfig(kdim=30, max_restarts=10, rtol=1e-6)
    # reference all-CPU
    R0 = ref.residual(q)
    bj_r = rnk.assemble_element_blocks(ref, q, shift)
    x_r, it_r, rr_r = rnk.gmres_solve(lambda v: rnk.jfnk_matvec(v, q, R0, ref.residual, shift), b, kc,
                                      precond=lambda v: rnk.ej_apply(bj_r, v))
    # reference host code, device matvec and preconditioner
    qd = torch.as_tensor(q, device="cuda")
    R0d = dev.residual(qd)
    bj_d = nk.assemble_element_blocks(dev, qd, shift)

    def matvec(v):
        return nk.jfnk_matvec(torch.as_tensor(v, device="cuda"), qd, R0d, dev.residual, shift).cpu().numpy()
    x_d, it_d, rr_d = rnk.gmres_solve(matvec, b, kc, precond=bj_d.apply)
    assert abs(it_d - it_r) <= 1 and rr_d <= 1e-6
    # two solves stopped at relres <= 1e-6 (FD matvecs carry 1e-10 noise):
    # the iterates agree to the solve tolerance
    assert _rel(x_d, x_r) <= 1e-5


def test_reference_ptc_with_device_stage_function_and_pmg(cuda):
    c = cases.config(1)
    dev = Discretization(c.mesh, c.p, c.eqn)
    s = ti.get_scheme("esdirk3")
    adt = s.a[1, 1] * c.dt
    R0 = dev.residual(c.q0)
    explicit = c.q0 + c.dt * s.a[1, 0] * R0

    def F(q):                               # the ESDIRK stage function on the device
        return (q - explicit) / adt - dev.residual(q)
    ctx = pmg.PmgContext(dev, pmg.PmgPrecondConfig(pmg.PHierarchy.parse("3-2", "2"), smoother_shift=50.0))

    def factory(q, dtau):
        ctx.prepare(q, 1.0 / adt + 1.0 / dtau)
        return ctx.precondition
    cfg = rnk.PtcConfig(dtau_init=c.dt, rtol=1e-4)
    kc = rnk.KrylovConfig(kdim=30, rtol=1e-3)
    q_r, st_r = rnk.ptc_solve(F, c.q0, cfg, kc, precond_factory=factory)
    # the re-hosted device PTC on the same problem
    ctx2 = pmg.PmgContext(dev, pmg.PmgPrecondConfig(pmg.PHierarchy.parse("3-2", "2"), smoother_shift=50.0))

    def factory2(q, dtau):
        ctx2.prepare(q, 1.0 / adt + 1.0 / dtau)
        return ctx2.precondition
    Fd = lambda q: torch.as_tensor(F(q.cpu().numpy()), device="cuda")  # noqa: E731
    q_d, st_d = nk.ptc_solve(Fd, torch.as_tensor(c.q0, device="cuda"), nk.PtcConfig(dtau_init=c.dt, rtol=1e-4),
                             nk.KrylovConfig(kdim=30, rtol=1e-3), precond_factory=factory2)
    assert st_r["converged"] and st_d["converged"]
    assert st_r["iters"] == st_d["iters"]
    assert abs(st_r["gmres_iters"] - st_d["gmres_iters"]) <= st_r["iters"]
    assert _rel(q_d, q_r) <= 1e-7
