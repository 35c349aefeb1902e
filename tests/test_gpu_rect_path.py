"""The axis-aligned-rectangle residual path (csrc/fr_rect.cu) against the
general bilinear kernels (csrc/fr_kernels.cu) and the oracle.

Every BASELINE mesh is made of axis-aligned rectangles, so the rectangle
kernels carry the headline numbers; the general kernels keep serving
curved / skewed meshes.  Both implement spatial.py:501-570: they must agree
to rounding on every kind, degree, boundary tag, option and fused
epilogue, and the rectangle path must be chosen exactly when the mesh
qualifies."""

import numpy as np
import pytest
import torch

from oracle.fr_oracle import OracleDisc
from paper_2202_09733_b200 import _lib, cases, mesh as mm
from paper_2202_09733_b200.equation import EquationSpec, NonPhysicalStateError
from paper_2202_09733_b200.spatial import Discretization

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    b = b.cpu().numpy() if isinstance(b, torch.Tensor) else b
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _both(d, fn):
    assert d.residual_path() == "rect"
    r = fn()
    d.residual_path("general")
    g = fn()
    d.residual_path("rect")
    return r, g


def test_path_selection():
    c = cases.config(1, nx=4)
    assert Discretization(c.mesh, 3, c.eqn).residual_path() == "rect"
    cyl = mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3)
    eq = EquationSpec(kind="navier-stokes", mach=0.3, reynolds=200.0)
    assert Discretization(cyl, 3, eq).residual_path() == "general"
    adv = EquationSpec(kind="advection-diffusion", advection=(1.0, 0.5), diffusivity=0.1)
    assert Discretization(c.mesh, 3, adv).residual_path() == "general"
    assert Discretization(c.mesh, 0, c.eqn).residual_path() == "general"


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("kind", ["euler", "navier-stokes"])
@pytest.mark.parametrize("opts", [{}, {"riemann": "rusanov", "viscous_scheme": "ldg"}])
def test_rect_matches_general_and_oracle(cuda, p, kind, opts):
    m = mm.generate_box(5, 4, 2.0, 1.5, periodic=True)
    eqn = EquationSpec(kind=kind, mach=0.4, reynolds=80.0, **opts)
    o = OracleDisc(m, p, eqn)
    rng = np.random.default_rng(p)
    q = o.free_stream_field() * (1 + 0.05 * rng.standard_normal(o.n_dofs))
    d = Discretization(m, p, eqn)
    qd = torch.as_tensor(q, device="cuda")
    r, g = _both(d, lambda: d.residual(qd))
    Ro = o.residual(q)
    assert _rel(r, Ro) <= 1e-12
    assert _rel(r, g) <= 1e-12


@pytest.mark.parametrize("tags", [("wall-adiabatic", "wall-slip"), ("wall-isothermal", "far-field"),
                                  ("far-field", "wall-adiabatic")])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_rect_channel_walls(cuda, tags, p):
    yn = np.array([0.0, 0.02, 0.07, 0.2, 0.45, 1.0])
    ch = mm.generate_channel(6, 5, 2.0, yn, bottom=tags[0], top=tags[1])
    eqn = EquationSpec(kind="navier-stokes", mach=0.3, reynolds=300.0, wall_temperature=1.1 / (1.4 * 0.09))
    o = OracleDisc(ch, p, eqn)
    q = o.free_stream_field() * (1 + 0.02 * np.random.default_rng(3).standard_normal(o.n_dofs))
    d = Discretization(ch, p, eqn)
    qd = torch.as_tensor(q, device="cuda")
    r, g = _both(d, lambda: d.residual(qd))
    assert _rel(r, o.residual(q)) <= 1e-12
    assert _rel(r, g) <= 1e-12


def test_rect_self_periodic_single_element(cuda):
    m = mm.generate_box(1, 1, 1.0, 1.0, periodic=True)
    eqn = EquationSpec(kind="navier-stokes", mach=0.3, reynolds=50.0)
    o = OracleDisc(m, 3, eqn)
    q = o.free_stream_field() * (1 + 0.02 * np.random.default_rng(4).standard_normal(o.n_dofs))
    d = Discretization(m, 3, eqn)
    assert d.residual_path() == "rect"
    assert _rel(d.residual(torch.as_tensor(q, device="cuda")), o.residual(q)) <= 1e-12


@pytest.mark.parametrize("mode", range(9))
def test_rect_epilogues_match_general(cuda, mode):
    c = cases.config(1, nx=6)
    d = Discretization(c.mesh, c.p, c.eqn)
    n = d.n_dofs
    gen = torch.Generator("cuda").manual_seed(mode)
    q = torch.as_tensor(c.q0, device="cuda")
    rnd = lambda: torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)  # noqa: E731
    X, R0, E, Sb, Se, Q0 = rnd(), rnd(), rnd(), rnd(), rnd(), rnd()
    lam = torch.rand(c.mesh.n_elements, dtype=torch.float64, device="cuda", generator=gen) + 0.5
    kw = dict(X=X if mode in (_lib.EPI_JV, _lib.EPI_STAGE_JV) else None, eps=1e-6, s=2.5, adt=0.3, dtau=0.7,
              R0=R0, E=E, Sb=Sb, Se=Se, Q0=Q0, dtau_e=lam, alpha=0.5)
    r, g = _both(d, lambda: d.eval(q, mode, **kw))
    # the Jv forms divide R rounding by eps: compare at the FD noise floor
    tol = 1e-8 if mode in (_lib.EPI_JV, _lib.EPI_STAGE_JV) else 1e-12
    assert _rel(r, g) <= tol


def test_rect_jv_bitwise_own_residual(cuda):
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    q = torch.as_tensor(c.q0, device="cuda")
    R0 = d.residual(q)
    v = torch.randn(d.n_dofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(9))
    out = d.eval(q, _lib.EPI_JV, X=v, eps=1e-6, s=3.7, R0=R0)
    qp = q + 1e-6 * v  # same rounding as the kernel's q + eps X
    ref = 3.7 * v - (d.residual(qp) - R0) / torch.full_like(R0, 1e-6)
    assert torch.equal(out, ref)


@pytest.mark.parametrize("kind", ["euler", "navier-stokes"])
@pytest.mark.parametrize("where", ["state", "trace"])
def test_rect_nonphysical_reports_smallest_element(cuda, kind, where):
    m = mm.generate_box(6, 5, 1.0, 1.0, periodic=True)
    eqn = EquationSpec(kind=kind, mach=0.3, reynolds=100.0)
    o = OracleDisc(m, 3, eqn)
    q = o.free_stream_field().copy().reshape(-1, 4, 4, 4)
    if where == "state":
        q[17, 2, 1, 0] = -1.0
        q[23, 0, 0, 0] = -1.0
    else:  # physical at the points, negative pressure on a face-1 trace
        q[11, 1, :, 3] = [q[11, 1, 0, 3]] * 3 + [0.6]
        q[19, 2, :, 3] = [q[19, 2, 0, 3]] * 3 + [0.6]
    d = Discretization(m, 3, eqn)
    assert d.residual_path() == "rect"
    with pytest.raises(NonPhysicalStateError) as ei:
        o.residual(q.reshape(-1))
    with pytest.raises(NonPhysicalStateError) as ed:
        d.residual(torch.as_tensor(q.reshape(-1), device="cuda"))
    assert ei.value.what == where
    assert (ed.value.element, ed.value.what) == (ei.value.element, ei.value.what)


def test_rect_config2_matches_general_full_size(cuda):
    c = cases.config(2)
    d = Discretization(c.mesh, c.p, c.eqn)
    q = torch.as_tensor(c.q0, device="cuda")
    r, g = _both(d, lambda: d.residual(q))
    assert _rel(r, g) <= 2e-9  # both within the reference's own floor of the truth (1.2e-9)
    assert torch.equal(r, d.residual(q)), "bitwise determinism"


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("kind", ["euler", "navier-stokes"])
def test_chain_variants_agree(cuda, p, kind):
    """The two rectangle chains -- k_rgf (k_rface for euler) + k_rasm with the
    common flux folded in ("rect", the default) and k_rface + k_rgrad + k_rfc +
    k_rasm ("rect4"; "rect" picks one per degree) -- evaluate the same formulas in the same order (the
    compiler's FMA contraction differs between the kernels, so they agree to
    rounding, not bit for bit): on walled channels (every boundary branch),
    with Rusanov / LDG, for R, the fused Jv and the defect epilogue; more
    element blocks than resident CTAs, element runs that end inside a CTA,
    neighbours inside and outside a CTA's run (the shared-memory trace
    hand-over)."""
    yn = np.array([0.0, 0.03, 0.1, 0.3, 0.6, 1.0])
    nx = 210 if p == 4 else 23
    for m, opts in ((mm.generate_channel(nx, 5, 2.0, yn, bottom="wall-isothermal", top="wall-adiabatic"), {}),
                    (mm.generate_channel(7, 5, 2.0, yn, bottom="far-field", top="wall-slip"), {}),
                    (mm.generate_box(9, 7, 2.0, 1.5, periodic=True),
                     {"riemann": "rusanov", "viscous_scheme": "ldg"})):
        eqn = EquationSpec(kind=kind, mach=0.3, reynolds=150.0, **opts)
        d = Discretization(m, p, eqn)
        n = d.n_dofs
        o = OracleDisc(m, p, eqn)
        q = torch.as_tensor(o.free_stream_field() * (1 + 0.03 * np.random.default_rng(p).standard_normal(n)),
                            device="cuda")
        X = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(p))
        out = {}
        for path in ("rect2", "rect4", "rect"):
            assert d.residual_path(path) == path
            out[path] = (d.residual(q), d.eval(q, _lib.EPI_JV, X=X, eps=1e-6, s=1.5, R0=X),
                         d.eval(q, _lib.EPI_DEFECT, s=2.0, Sb=X, Se=0.25))
        assert _rel(out["rect2"][0], out["rect4"][0]) <= 1e-13
        assert _rel(out["rect2"][1], out["rect4"][1]) <= 1e-8   # rounding / eps
        assert _rel(out["rect2"][2], out["rect4"][2]) <= 1e-13
        # the default is one of the two, bit for bit (the four-kernel chain at p = 2)
        same = out["rect4"] if p == 2 else out["rect2"]
        assert all(torch.equal(a, b) for a, b in zip(out["rect"], same))


def _renumber(mesh, perm):
    """The same mesh with element e renamed perm[e] (face roles L / R kept)."""
    M = mesh.n_elements
    inv = np.empty(M, dtype=np.int64)
    inv[perm] = np.arange(M)
    elements = mesh.elements[inv]
    itf = mesh.interior_faces.copy()
    itf[:, 0], itf[:, 2] = perm[itf[:, 0]], perm[itf[:, 2]]
    itf = itf[np.lexsort((itf[:, 1], itf[:, 0]))]
    bf = mesh.boundary_faces.copy()
    bf[:, 0] = perm[bf[:, 0]]
    order = np.lexsort((bf[:, 1], bf[:, 0]))
    tags = tuple(mesh.boundary_tags[i] for i in order)
    return mm.Mesh(mesh.nodes, elements, itf, bf[order], tags)


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_arbitrary_element_numbering(cuda, p):
    """The rectangle kernels take the connectivity as a gathered list (the
    reference's face batches, spatial.py:521-526), not a structured grid: a
    random renumbering of the elements scatters every CTA's element run over
    the mesh -- neighbours inside and outside a CTA's run in every pattern, the
    shared-memory trace hand-over on arbitrary pairs, self-neighbours through
    the periodic wrap -- and must give the same R (against the oracle on the
    renumbered mesh, and the renumbered result of the ordered mesh bit for
    bit: the per-element arithmetic does not depend on the numbering)."""
    yn = np.array([0.0, 0.02, 0.07, 0.2, 0.45, 0.7, 1.0])
    rng = np.random.default_rng(40 + p)
    for m0 in (mm.generate_channel(29, 6, 3.0, yn, bottom="wall-isothermal", top="wall-adiabatic"),
               mm.generate_box(13, 11, 2.0, 1.5, periodic=True),
               mm.generate_box(1, 7, 1.0, 3.0, periodic=True)):
        M = m0.n_elements
        perm = rng.permutation(M)
        m1 = _renumber(m0, perm)
        eqn = EquationSpec(kind="navier-stokes", mach=0.3, reynolds=150.0)
        d0, d1 = Discretization(m0, p, eqn), Discretization(m1, p, eqn)
        assert d0.residual_path() == "rect" and d1.residual_path() == "rect"
        o1 = OracleDisc(m1, p, eqn)
        npe = d0.n_dofs // M
        q0 = o1.free_stream_field() * (1 + 0.03 * rng.standard_normal(d0.n_dofs))
        q1 = np.empty_like(q0)
        q1.reshape(M, npe)[perm] = q0.reshape(M, npe)
        X0 = rng.standard_normal(d0.n_dofs)
        X1 = np.empty_like(X0)
        X1.reshape(M, npe)[perm] = X0.reshape(M, npe)
        t = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
        for path in ("rect2", "rect4", "rect"):
            d0.residual_path(path), d1.residual_path(path)
            R0, R1 = d0.residual(t(q0)), d1.residual(t(q1))
            assert _rel(R1, o1.residual(q1)) <= 1e-12
            assert torch.equal(R1.view(M, npe)[t(perm)], R0.view(M, npe))
            J0 = d0.eval(t(q0), _lib.EPI_JV, X=t(X0), eps=1e-6, s=1.5, R0=R0)
            J1 = d1.eval(t(q1), _lib.EPI_JV, X=t(X1), eps=1e-6, s=1.5, R0=R1)
            assert torch.equal(J1.view(M, npe)[t(perm)], J0.view(M, npe))


def test_misaligned_operands_are_rejected(cuda):
    """The rectangle kernels move whole points (4 doubles, 256-bit accesses): an
    array that does not start on a 32-byte boundary is refused with a clear
    error instead of faulting."""
    c = cases.config(1, nx=4)
    d = Discretization(c.mesh, c.p, c.eqn)
    n = d.n_dofs
    buf = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    q = torch.as_tensor(c.q0, device="cuda")
    buf[1:].copy_(q)
    with pytest.raises(_lib.PmgbError, match="32-byte aligned"):
        d.residual(buf[1:])
    with pytest.raises(_lib.PmgbError, match="32-byte aligned"):
        d.eval(q, _lib.EPI_JV, X=buf[1:], eps=1e-6, s=1.0, R0=q)
