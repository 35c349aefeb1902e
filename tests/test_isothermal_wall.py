"""No-slip isothermal wall ("wall-isothermal", BASELINE config 4).

Not in the reference (its wall tags are wall-adiabatic / wall-slip /
far-field, spatial.py:183-203), so parity is against the oracle
restatement only (OracleDisc._w_out): the inviscid ghost is the mirrored
no-slip state of the adiabatic wall (spatial.py:198-203), the BR1 ghost of
the viscous variables carries T = 2 T_w - T so the common value holds
T = T_w, and the wall's energy viscous flux is kept (the adiabatic wall
zeroes it, spatial.py:566-567).  CPU tests pin the oracle by property;
GPU tests compare the device path with it at the 1e-12 residual bar.
"""

import numpy as np
import pytest
import torch

from oracle import solver_oracle as so
from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import mesh as mm
from paper_2202_09733_b200.equation import EquationSpec

YN = np.array([0.0, 0.05, 0.2, 0.5, 1.0])


def _chan(bottom="wall-isothermal", top="wall-slip"):
    return mm.generate_channel(6, 4, 2.0, YN, bottom=bottom, top=top)


def _eqn(tw_factor=1.2, **kw):
    base = EquationSpec(kind="navier-stokes", mach=0.3, reynolds=200.0, **kw)
    return EquationSpec(kind="navier-stokes", mach=0.3, reynolds=200.0,
                        wall_temperature=tw_factor * base.t_wall, **kw)


def _rest(orc, T):
    """Fluid at rest, uniform density 1 and temperature T = p / rho."""
    q = orc.free_stream_field().reshape(-1, 4).copy()
    q[:, 1:3] = 0.0
    q[:, 3] = T / (orc.eqn.gamma - 1.0)
    return q.reshape(-1)


def _state(orc, seed=1):
    q = orc.free_stream_field()
    return q * (1.0 + 0.01 * np.random.default_rng(seed).standard_normal(q.shape))


def test_rest_state_at_wall_temperature_is_steady():
    eqn = _eqn(1.0)
    for p in (1, 3):
        o = OracleDisc(_chan("wall-isothermal", "wall-isothermal"), p, eqn)
        assert np.max(np.abs(o.residual(_rest(o, eqn.t_wall)))) <= 1e-11


def test_hot_wall_heats_and_cold_wall_cools_the_fluid():
    for factor, sign in ((1.5, 1.0), (0.7, -1.0)):
        eqn = _eqn(factor)
        o = OracleDisc(_chan(), 2, eqn)
        T_inf = EquationSpec(kind="navier-stokes", mach=0.3, reynolds=200.0).t_wall
        R = o.residual(_rest(o, T_inf)).reshape(-1, 9, 4)
        wall_cells = np.arange(6)                    # bottom row, face 0 on the wall
        dE = R[wall_cells, :, 3].sum()
        assert sign * dE > 0.0
        assert np.max(np.abs(R[:, :, 0:3])) <= 1e-10                 # anywhere


def test_isothermal_equals_adiabatic_for_euler_and_inviscid_part():
    e = EquationSpec(kind="euler", mach=0.3)
    oa, oi = OracleDisc(_chan("wall-adiabatic"), 2, e), OracleDisc(_chan(), 2, e)
    q = _state(oa)
    assert np.array_equal(oa.residual(q), oi.residual(q))


def test_wall_temperature_validation_and_default():
    with pytest.raises(ValueError, match="wall temperature"):
        EquationSpec(kind="navier-stokes", mach=0.3, reynolds=100.0, wall_temperature=-1.0)
    e = EquationSpec(kind="navier-stokes", mach=0.5, reynolds=100.0)
    assert e.t_wall == pytest.approx(1.0 / (1.4 * 0.25))


# --------------------------------------------------------------------- GPU

def _t(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def _rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


MESHES = {
    "chan": lambda: _chan(),
    "chan2": lambda: _chan("wall-isothermal", "wall-isothermal"),
    "cyl": lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3, wall_tag="wall-isothermal"),
}


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", [("roe", "br1"), ("rusanov", "ldg")])
@pytest.mark.parametrize("mesh", list(MESHES))
def test_device_residual_matches_oracle(cuda, mesh, scheme):
    from paper_2202_09733_b200.spatial import Discretization
    eqn = _eqn(1.2, riemann=scheme[0], viscous_scheme=scheme[1])
    m = MESHES[mesh]()
    for p in (1, 2, 3, 4, 5):
        o, d = OracleDisc(m, p, eqn), Discretization(m, p, eqn)
        q = _state(o)
        assert _rel(d.residual(q), o.residual(q)) <= 1e-12, (mesh, p)


@pytest.mark.gpu
def test_device_rest_state_steady_and_local_equals_global(cuda):
    from paper_2202_09733_b200.spatial import Discretization
    eqn = _eqn(1.0)
    m = MESHES["chan2"]()
    o, d = OracleDisc(m, 3, eqn), Discretization(m, 3, eqn)
    assert np.max(np.abs(d.residual(_rest(o, eqn.t_wall)))) <= 1e-11
    eqn = _eqn(1.3)
    o, d = OracleDisc(m, 2, eqn), Discretization(m, 2, eqn)
    q = _state(o)
    fo, fd = o.freeze(q), d.freeze(q)
    R = d.residual(q)
    for e in (0, 3, 5, m.n_elements - 1):               # bottom and top wall rows
        Q = q[o.offsets[e]:o.offsets[e + 1]].reshape(3, 3, 4)
        B = np.stack([Q, Q * 1.001, Q * 0.999])
        assert _rel(d.element_residual(e, B, fd), o.element_residual(e, B, fo)) <= 1e-12, e
        Re = d.element_residual(e, Q, fd)
        assert np.max(np.abs(Re.reshape(-1) - R[o.offsets[e]:o.offsets[e + 1]])) <= 1e-12


@pytest.mark.gpu
def test_device_blocks_sparse_and_forces_match_oracle(cuda):
    from paper_2202_09733_b200 import newton_krylov as nk
    from paper_2202_09733_b200.spatial import Discretization
    eqn = _eqn(1.2)
    m = MESHES["chan"]()
    o, d = OracleDisc(m, 2, eqn), Discretization(m, 2, eqn)
    q = _state(o)
    ob = so.assemble_blocks(o, q, 30.0)
    db = nk.assemble_element_blocks(d, _t(q), 30.0)
    assert _rel(db.inv[0], ob.inv) <= 1e-8
    A = nk.assemble_sparse_blocks(d, _t(q), 30.0)
    S = so.assemble_sparse(o, q, 30.0)
    assert np.array_equal(A.indices, S.indices)
    assert _rel(A.blocks, np.stack(S.blocks)) <= 1e-7
    assert np.allclose(d.compute_forces(q), o.compute_forces(q), rtol=1e-12, atol=1e-14)
