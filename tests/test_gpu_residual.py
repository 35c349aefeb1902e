"""Device FR residual / freeze / element-local residual vs the oracle.

Tolerance: max|R_gpu - R_oracle| <= 1e-12 max|R_oracle| (north star; the
measured different-rounding floor is 1.5e-13)."""

import numpy as np
import pytest
import torch

from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import cases, mesh as mm
from paper_2202_09733_b200.equation import EquationSpec, NonPhysicalStateError
from paper_2202_09733_b200.spatial import Discretization

pytestmark = pytest.mark.gpu

RTOL = 1e-12

MESHES = {
    "box4p": lambda: mm.generate_box(4, 4, 1.0, 1.0, periodic=True),
    "box3ff": lambda: mm.generate_box(3, 3, 2.0, 1.5),
    "cyl_adiab": lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3),
    "cyl_slip": lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3, wall_tag="wall-slip"),
    "box1p": lambda: mm.generate_box(1, 1, 1.0, 1.0, periodic=True),
    "chan": lambda: mm.generate_channel(6, 4, 2.0, np.array([0.0, 0.05, 0.2, 0.5, 1.0])),
}

KINDS = {
    "euler": dict(kind="euler", mach=0.3),
    "ns": dict(kind="navier-stokes", mach=0.3, reynolds=200.0),
    "adv": dict(kind="advection-diffusion", advection=(0.7, 0.4)),
    "advd": dict(kind="advection-diffusion", advection=(0.7, 0.4), diffusivity=0.02),
}


def _state(orc, kind, seed=1):
    rng = np.random.default_rng(seed)
    if orc.eqn.kind == "advection-diffusion":
        return rng.standard_normal(orc.n_dofs)
    q = orc.free_stream_field()
    return q * (1.0 + 0.01 * rng.standard_normal(q.shape))


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("kind", list(KINDS))
@pytest.mark.parametrize("p", [0, 1, 2, 3, 4, 5])
def test_residual_matches_oracle_periodic(cuda, kind, p):
    m = MESHES["box4p"]()
    eqn = EquationSpec(**KINDS[kind])
    orc = OracleDisc(m, p, eqn)
    dev = Discretization(m, p, eqn)
    q = _state(orc, kind)
    assert _rel(dev.residual(q), orc.residual(q)) <= RTOL


@pytest.mark.parametrize("mesh", ["box3ff", "cyl_adiab", "cyl_slip", "box1p", "chan"])
@pytest.mark.parametrize("kind", list(KINDS))
def test_residual_matches_oracle_boundaries(cuda, mesh, kind):
    m = MESHES[mesh]()
    eqn = EquationSpec(**KINDS[kind])
    for p in (2, 3):
        orc = OracleDisc(m, p, eqn)
        dev = Discretization(m, p, eqn)
        q = _state(orc, kind)
        assert _rel(dev.residual(q), orc.residual(q)) <= RTOL, (mesh, kind, p)


def test_config1_residual(cuda):
    c = cases.config(1)
    orc = OracleDisc(c.mesh, c.p, c.eqn)
    dev = Discretization(c.mesh, c.p, c.eqn)
    assert _rel(dev.residual(c.q0), orc.residual(c.q0)) <= RTOL


def test_tensor_in_tensor_out_and_deterministic(cuda):
    c = cases.config(1)
    dev = Discretization(c.mesh, c.p, c.eqn)
    q = torch.as_tensor(c.q0, device=cuda)
    R1 = dev.residual(q)
    R2 = dev.residual(q)
    assert isinstance(R1, torch.Tensor) and R1.is_cuda
    assert torch.equal(R1, R2)


@pytest.mark.parametrize("kind", ["euler", "ns"])
def test_free_stream_preserved(cuda, kind):
    eqn = EquationSpec(**KINDS[kind])
    for name in ("box3ff", "box4p"):
        m = MESHES[name]()
        for p in (1, 2, 3, 4):
            dev = Discretization(m, p, eqn)
            R = dev.residual(dev.free_stream_field().data)
            assert float(R.abs().max()) <= 1e-11


def test_nonphysical_reports_smallest_element(cuda):
    m = mm.generate_box(2, 2, 1.0, 1.0, periodic=True)
    eqn = EquationSpec(kind="euler", mach=0.3)
    dev = Discretization(m, 1, eqn)
    f = dev.free_stream_field()
    f.element(3)[..., 0] = -1.0
    f.element(2)[..., 3] = -5.0
    with pytest.raises(NonPhysicalStateError) as err:
        dev.residual(f.data)
    assert err.value.element == 2
    # the status word is cleared: a good state evaluates again
    dev.residual(dev.free_stream_field().data)


@pytest.mark.parametrize("kind", ["euler", "ns", "advd"])
@pytest.mark.parametrize("mesh", ["box4p", "cyl_adiab", "chan"])
def test_element_residual_matches_oracle(cuda, kind, mesh):
    m = MESHES[mesh]()
    eqn = EquationSpec(**KINDS[kind])
    p = 2
    orc = OracleDisc(m, p, eqn)
    dev = Discretization(m, p, eqn)
    q = _state(orc, kind)
    fo = orc.freeze(q)
    fd = dev.freeze(q)
    n, nv = p + 1, eqn.nvars
    for e in (0, 3, m.n_elements - 1):
        Q = q[orc.offsets[e]:orc.offsets[e + 1]].reshape(n, n, nv)
        B = np.stack([Q, Q * 1.001, Q * 0.999])
        ref = orc.element_residual(e, B, fo)
        got = dev.element_residual(e, B, fd)
        assert _rel(got, ref) <= RTOL, e


def test_local_equals_global(cuda):
    # reference tests/test_spatial.py:296-307
    m = MESHES["box4p"]()
    eqn = EquationSpec(**KINDS["ns"])
    dev = Discretization(m, 2, eqn)
    orc = OracleDisc(m, 2, eqn)
    q = _state(orc, "ns")
    R = dev.residual(q)
    fr = dev.freeze(q)
    for e in (0, 4, 7):
        Re = dev.element_residual(e, q[orc.offsets[e]:orc.offsets[e + 1]].reshape(3, 3, 4), fr)
        assert np.max(np.abs(Re.reshape(-1) - R[orc.offsets[e]:orc.offsets[e + 1]])) <= 1e-12


def test_residual_batch_host_pipeline(cuda):
    c = cases.config(1)
    dev = Discretization(c.mesh, c.p, c.eqn)
    rng = np.random.default_rng(3)
    qs = [c.q0 * (1.0 + 1e-3 * rng.standard_normal(c.q0.shape)) for _ in range(5)]
    outs = dev.residual_batch([torch.from_numpy(q).pin_memory() for q in qs])
    for q, R in zip(qs, outs):
        assert np.array_equal(R.numpy(), dev.residual(q))


# ---------------------------------------------------------------------------
# BASELINE interface options (Rusanov flux, LDG viscous scheme): not in the
# reference, pinned to the oracle restatement (fr_oracle.rusanov_flux,
# OracleDisc._common_w / _common_fv) at the same 1e-12 bar

SCHEMES = [("rusanov", "br1"), ("roe", "ldg"), ("rusanov", "ldg")]


@pytest.mark.parametrize("riemann,visc", SCHEMES)
@pytest.mark.parametrize("kind", ["euler", "ns", "advd"])
@pytest.mark.parametrize("mesh", ["box4p", "box3ff", "cyl_adiab", "cyl_slip", "chan", "box1p"])
def test_residual_options_match_oracle(cuda, riemann, visc, kind, mesh):
    m = MESHES[mesh]()
    eqn = EquationSpec(**KINDS[kind], riemann=riemann, viscous_scheme=visc)
    for p in (1, 3, 4):
        orc = OracleDisc(m, p, eqn)
        dev = Discretization(m, p, eqn)
        q = _state(orc, kind)
        assert _rel(dev.residual(q), orc.residual(q)) <= RTOL, (mesh, kind, p)


@pytest.mark.parametrize("riemann,visc", SCHEMES)
@pytest.mark.parametrize("mesh", ["box4p", "cyl_adiab", "chan"])
def test_element_residual_options_match_oracle(cuda, riemann, visc, mesh):
    m = MESHES[mesh]()
    eqn = EquationSpec(**KINDS["ns"], riemann=riemann, viscous_scheme=visc)
    p = 2
    orc = OracleDisc(m, p, eqn)
    dev = Discretization(m, p, eqn)
    q = _state(orc, "ns")
    fo, fd = orc.freeze(q), dev.freeze(q)
    R = dev.residual(q)
    for e in (0, 3, m.n_elements - 1):
        Q = q[orc.offsets[e]:orc.offsets[e + 1]].reshape(3, 3, 4)
        B = np.stack([Q, Q * 1.001, Q * 0.999])
        assert _rel(dev.element_residual(e, B, fd), orc.element_residual(e, B, fo)) <= RTOL, e
        # local == global holds for every interface scheme
        Re = dev.element_residual(e, Q, fd)
        assert np.max(np.abs(Re.reshape(-1) - R[orc.offsets[e]:orc.offsets[e + 1]])) <= 1e-12


@pytest.mark.parametrize("riemann,visc", SCHEMES)
def test_free_stream_preserved_options(cuda, riemann, visc):
    eqn = EquationSpec(**KINDS["ns"], riemann=riemann, viscous_scheme=visc)
    for mesh in ("box4p", "box3ff"):   # periodic and far-field (walls are not free-stream steady)
        m = MESHES[mesh]()
        dev = Discretization(m, 3, eqn)
        q = OracleDisc(m, 3, eqn).free_stream_field()
        assert np.max(np.abs(dev.residual(q))) <= 1e-11


def test_epilogue_specialization_is_bitwise(cuda):
    # the assemble kernels' compile-time epilogue instantiations (R, Jv, PTC
    # Jv, defect, F at their own register targets; async at p=4, plain at
    # p=2) must give the runtime-switch kernels' bits in every mode
    import os
    import subprocess
    import sys
    from pathlib import Path
    script = str(Path(__file__).parent / "_epi_modes_digest.py")
    runs = []
    for flag in ("1", "0"):
        env = dict(os.environ, PMGB_EPI_SPECIALIZE=flag)
        r = subprocess.run([sys.executable, script], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        runs.append(r.stdout.split())
    assert len(runs[0]) == 16 and runs[0] == runs[1]
