"""Wall forces (compute_forces, spatial.py:633-695) against goldens from the
reference (tests/golden/make_golden_forces.py): the oracle on the CPU, the
device path through pmgb_wall_forces on the GPU."""

from pathlib import Path

import numpy as np
import pytest

from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import cases, mesh as mm
from paper_2202_09733_b200.equation import EquationSpec

G = np.load(Path(__file__).parent / "golden" / "golden_forces.npz")
CASES = {
    "cyl_ns2": (lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3),
                EquationSpec(kind="navier-stokes", mach=0.3, reynolds=200.0), 2),
    "cyl_slip_euler2": (lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3, wall_tag="wall-slip"),
                        EquationSpec(kind="euler", mach=0.3), 2),
    "chan_ns3": (lambda: cases.config(4, nx=16).mesh, cases.config(4, nx=16).eqn, 3),
}


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_forces_match_reference(name):
    mk, eqn, p = CASES[name]
    o = OracleDisc(mk(), p, eqn)
    assert np.allclose(o.compute_forces(G[f"{name}/q"]), G[f"{name}/F"], rtol=1e-12, atol=1e-14)


def test_oracle_forces_errors():
    with pytest.raises(ValueError, match="no wall"):
        OracleDisc(mm.generate_box(2, 2, 1.0, 1.0, periodic=True), 1,
                   EquationSpec(kind="euler", mach=0.3)).compute_forces(np.ones(64))


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_device_forces_match_reference(cuda, name):
    from paper_2202_09733_b200.spatial import Discretization
    mk, eqn, p = CASES[name]
    d = Discretization(mk(), p, eqn)
    assert np.allclose(d.compute_forces(G[f"{name}/q"]), G[f"{name}/F"], rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
def test_device_forces_errors(cuda):
    from paper_2202_09733_b200.spatial import Discretization
    d = Discretization(mm.generate_box(2, 2, 1.0, 1.0, periodic=True), 1, EquationSpec(kind="euler", mach=0.3))
    with pytest.raises(ValueError, match="no wall"):
        d.compute_forces(d.free_stream_field().data)
    d2 = Discretization(mm.generate_box(2, 2, 1.0, 1.0), 1,
                        EquationSpec(kind="advection-diffusion", advection=(1.0, 0.0), diffusivity=0.1))
    with pytest.raises(ValueError, match="flow equations"):
        d2.compute_forces(d2.free_stream_field().data)
