"""Mixed-degree / p-adaptive FR against the REFERENCE's
own outputs on mixed degree maps (tests/golden/make_golden_mixed.py):

* host: p_adapt.nest_hierarchy (p_adapt.py:106-123) and one adapt event
  (:71-103, indicator + L2 projection / embedding transfer);
* device (csrc/fr_mixed.cu through pmgb_mdisc_*): R (spatial.py:501-570
  with the mortar faces of :468-497, :572-585), the frozen neighbour
  records of freeze (:700-766) and element_residual (:768-853) on a
  periodic box (degrees 1..5), a far-field box (with a p = 0 element), a
  stretched walled channel and a curved O-grid, Euler and Navier-Stokes:
  <= 1e-12 relative (max-norm).
"""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2202_09733_b200 import p_adapt

G = np.load(Path(__file__).parent / "golden" / "golden_mixed.npz")
MESHES = ("boxp", "boxff", "chan", "cyl")


def _rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_nest_hierarchy_matches_reference():
    got = []
    for levels in ((4, 2), (4, 3, 2, 1, 0), (5, 4), (3, 2, 1)):
        for p_e in range(levels[0] + 1):
            got.append(list(p_adapt.nest_hierarchy(p_e, levels[0], levels)) + [-1] * (5 - len(levels)))
    assert np.array_equal(np.array(got), G["nest/table"])
    with pytest.raises(ValueError):
        p_adapt.nest_hierarchy(3, 4, (4, 4))


def test_adapt_event_matches_reference():
    cfg = p_adapt.AdaptConfig(variable="momentum-x", nu_max=0.2, nu_min=0.001, p_min=1, p_max=4)
    new, deg, eta = p_adapt.adapt(G["adapt/q"], np.full(16, 3), 4, cfg)
    assert np.array_equal(deg, G["adapt/degrees"])
    assert np.allclose(eta, G["adapt/eta"], rtol=1e-12, atol=1e-15)
    assert _rel(new, G["adapt/q_new"]) <= 1e-13


def _disc(mname, kname):
    from paper_2202_09733_b200.equation import EquationSpec
    from paper_2202_09733_b200.mesh import build_mesh, generate_box, generate_cylinder_omesh
    from paper_2202_09733_b200.spatial import Discretization
    if mname == "boxp":
        m = generate_box(5, 4, 2.0, 1.5, periodic=True)
    elif mname == "boxff":
        m = generate_box(4, 4, 2.0, 2.0)
    elif mname == "cyl":
        m = generate_cylinder_omesh(12, 3, 0.5, 6.0, 1.3)
    else:
        yn = np.array([0.0, 0.03, 0.1, 0.25, 0.5, 1.0])
        nx = 5
        X, Y = np.meshgrid(np.linspace(0.0, 2.0, nx + 1), yn)
        nodes = np.stack([X.ravel(), Y.ravel()], axis=1)
        jj, ii = np.meshgrid(np.arange(5), np.arange(nx), indexing="ij")
        base = (jj * (nx + 1) + ii).ravel()
        elements = np.stack([base, base + 1, base + nx + 2, base + nx + 1], axis=1)
        eid = lambda i, j: j * nx + i  # noqa: E731
        bnd = {(eid(i, 0), 0): "wall-adiabatic" for i in range(nx)}
        bnd.update({(eid(i, 4), 2): "wall-slip" for i in range(nx)})
        m = build_mesh(nodes, elements, bnd, [(eid(nx - 1, j), 1, eid(0, j), 3) for j in range(5)])
    kw = dict(kind="euler", mach=0.3) if kname == "euler" else dict(kind="navier-stokes", mach=0.3, reynolds=150.0)
    d = Discretization(m, G[f"{mname}/{kname}/degrees"], EquationSpec(**kw))
    return m, d


@pytest.mark.gpu
@pytest.mark.parametrize("mname", MESHES)
@pytest.mark.parametrize("kname", ["euler", "ns"])
def test_mixed_residual_freeze_local_match_reference(cuda, mname, kname):
    from paper_2202_09733_b200.spatial import MixedDiscretization
    m, d = _disc(mname, kname)
    assert isinstance(d, MixedDiscretization)
    key = f"{mname}/{kname}"
    q = G[f"{key}/q"]
    R = d.residual(torch.as_tensor(q, device="cuda"))
    assert _rel(R, G[f"{key}/R"]) <= 1e-12
    assert np.array_equal(d.residual(q), R.cpu().numpy())   # NumPy in/out, bitwise the same
    fr = d.freeze(q)
    interior = np.array([[lk >= 0 for lk in row] for row in d._links[..., 0]])
    for name, got in (("rq", fr.rq), ("rw", fr.rw), ("rf", fr.rf)):
        if kname == "euler" and name != "rq":
            continue
        ref = G[f"{key}/{name}"][interior]
        assert _rel(got.cpu().numpy()[interior], ref) <= 1e-12, name
    for e in (0, 1, m.n_elements - 1):
        Q = G[f"{key}/local/e{e}/Q"]
        assert _rel(d.element_residual(e, Q, fr), G[f"{key}/local/e{e}/R"]) <= 1e-12, e
