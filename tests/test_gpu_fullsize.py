"""Device residual at the BASELINE.json full sizes, checked through
size-independent properties (the oracle is too slow at these sizes:
1.2 s per R at config 2, 28 s at config 5 on one core):

* free-stream preservation on periodic meshes (reference
  tests/test_spatial.py:112-132)
* discrete conservation on periodic meshes: sum_e sum_ab w_a w_b det R = 0
  (tests/test_spatial.py:135-176)
* bitwise determinism of repeated evaluations (tests/test_acceptance.py:472-501)
* element-local residual with frozen neighbours == global residual on
  sampled elements (tests/test_spatial.py:296-307); the local path
  evaluates gradients in a different arithmetic order, so the two agree to
  rounding, not bitwise
* Jv linear in X up to the FD truncation: Jv(2X) ~ 2 Jv(X)

Tolerances are in units of the rounding bound of one FR derivative of the
flux: TOL_EPS * (|E| + p)_inf * n^2 / h_min, i.e. ~18 ulp of the largest
flux times the derivative operator's norm.  Measured on B200: free stream
3.4e-12 (config 2) / 5.1e-11 (config 5); local vs global 4.4e-12 / 2.2e-10.
Conservation is bounded relative to the weighted sum of |R| with sqrt(M)
growth (per-element rounding errors add like a random walk).
"""

import numpy as np
import pytest
import torch

from paper_2202_09733_b200 import cases, newton_krylov as nk
from paper_2202_09733_b200.mesh import element_geometry
from paper_2202_09733_b200.operators import gauss_rule
from paper_2202_09733_b200.spatial import Discretization

pytestmark = pytest.mark.gpu
TOL_EPS = 4e-15


def _round_scale(c):
    fs = c.eqn.free_stream()
    g = c.eqn.gamma
    rho, u, v, E = fs
    p = (g - 1.0) * (E - 0.5 * (u * u + v * v) / rho)
    return (abs(E) + abs(p)) * (c.p + 1) ** 2 / c.mesh.h_min


def _weighted_sums(c, disc, R):
    n, nv = disc.n, disc.nvars
    w = gauss_rule(n)[1]
    det = element_geometry(c.mesh, c.p).det.reshape(-1, n, n)
    Rr = R.reshape(-1, n, n, nv)
    tot = np.einsum("a,b,mab,mabv->v", w, w, det, Rr)
    mag = np.einsum("a,b,mab,mabv->v", w, w, det, np.abs(Rr))
    return tot, mag


@pytest.mark.parametrize("k", [2, 4, 5])
def test_fullsize_properties(cuda, k):
    c = cases.config(k)
    d = Discretization(c.mesh, c.p, c.eqn)
    tol = TOL_EPS * _round_scale(c)
    periodic = k != 4  # config 4 has no-slip walls: free stream is not steady
    if periodic:
        Rf = d.residual(d.free_stream_field().data)
        assert float(Rf.abs().max()) <= tol, "free-stream preservation"
        del Rf
    q = torch.as_tensor(c.q0, device="cuda")
    R = d.residual(q)
    assert bool(torch.isfinite(R).all())
    assert torch.equal(R, d.residual(q)), "bitwise determinism"

    fr = d.freeze(q)
    M = c.mesh.n_elements
    elems = np.unique(np.concatenate([[0, 1, M - 1], np.random.default_rng(0).integers(0, M, 125)]))
    sz = d.elem_size
    Q = torch.stack([q[e * sz:(e + 1) * sz] for e in elems]).reshape(len(elems), d.n, d.n, d.nvars)
    Rl = d.element_residual(elems, Q, fr).reshape(len(elems), sz)
    Rg = torch.stack([R[e * sz:(e + 1) * sz] for e in elems])
    assert float((Rl - Rg).abs().max()) <= 2 * tol, "element-local == global"

    if periodic:
        tot, mag = _weighted_sums(c, d, R.cpu().numpy())
        # per-element rounding adds up like a random walk: ~sqrt(M) growth
        # (measured at config 5, M = 2^20: |sum| / sum|.| = 2.8e-12)
        bound = 1e-14 * np.sqrt(M) * np.maximum(mag, 1.0)
        assert np.all(np.abs(tot) <= bound), f"discrete conservation {tot} {mag}"

    if k == 2:
        X = torch.randn(d.n_dofs, dtype=torch.float64, device="cuda",
                        generator=torch.Generator("cuda").manual_seed(1))
        X = X / X.norm()
        J1 = nk.jfnk_matvec(X, q, R, d.residual, 3.0)
        J2 = nk.jfnk_matvec(2.0 * X, q, R, d.residual, 3.0)
        assert float((J2 - 2.0 * J1).norm() / J1.norm()) <= 1e-4  # O(eps |X|), eps = 1e-6


def test_fullsize_jv_bitwise_deterministic(cuda):
    # the fused Jv reads k_trace's q + eps X in k_fvn / k_assemble, which run
    # under programmatic dependent launch: those reads must follow the
    # dependency wait (a read-before-write race made steps nondeterministic)
    from paper_2202_09733_b200 import _lib
    c = cases.config(2)
    d = Discretization(c.mesh, c.p, c.eqn)
    q = torch.as_tensor(c.q0, device="cuda")
    R0 = d.residual(q)
    X = torch.randn(d.n_dofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    outs = [torch.empty_like(q) for _ in range(12)]
    for o in outs:
        d.eval(q, _lib.EPI_JV, o, X=X, eps=1e-6, s=2.5, R0=R0)
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("world", [1, 2, 4])
def test_slab_partition_owned_residual_bitwise(cuda, world):
    # the multi-GPU path's strips (owned rows + 2 halo rows) reproduce the
    # global residual on their owned rows bit for bit (one process, ranks
    # simulated, halos filled from the global field)
    from paper_2202_09733_b200.partition import PartitionedResidual, SlabPartition
    c = cases.config(2, nx=32)
    d = Discretization(c.mesh, c.p, c.eqn)
    q = torch.as_tensor(c.q0, device="cuda")
    Rg = d.residual(q).reshape(-1, d.elem_size)
    for rank in range(world):
        part = SlabPartition(32, 32, 10.0, 10.0, world, rank)
        pr = PartitionedResidual(part, c.p, c.eqn)
        pr.q_local.copy_(part.scatter_global(q, d.elem_size))
        Rl = pr.disc.residual(pr.q_local).reshape(-1, d.elem_size)
        own = torch.as_tensor(part.global_elements[part.owned], device="cuda")
        assert torch.equal(Rl[part.owned], Rg[own]), rank
