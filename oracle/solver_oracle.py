"""ORACLE (test infrastructure only).  NumPy restatement of the
reference's JFNK / EJ / pMG / stepper control flow on top of
``fr_oracle.OracleDisc``; used by tests/ as the parity checker and by
bench.py as the CPU baseline ("port") and the reference arm.

Citations (/root/reference/pkg/src/pmgflow/):
  newton_krylov.py: FD_EPS 25, ser_update 56-68, jfnk_matvec 71-76,
    gmres_solve 79-151, element_jacobian_block 174-184,
    assemble_element_blocks 187-210, BlockJacobian.apply 166-171,
    ptc_solve 377-437
  pmg.py: PmgPrecondConfig 72-86, _restrict/_prolong 117-136,
    LevelState 142-159, smooth_ej 162-164, PmgContext 181-298,
    pmg_solve 308-374
  time_integration.py: stage_function 138-141, esdirk_step 144-168,
    row_step 171-197
  harness.py: ImplicitDriver 277-369
"""

from __future__ import annotations

import numpy as np

from paper_2202_09733_b200.equation import NonPhysicalStateError
from paper_2202_09733_b200.operators import transfer_operators

from .fr_oracle import OracleDisc

FD_EPS = 1e-6


def ser_update(dtau, f_old, f_new, dtau_max, as_printed=False):
    if f_old == 0.0 or f_new == 0.0:
        return dtau_max
    r = (f_new / f_old) if as_printed else (f_old / f_new)
    return min(dtau * r, dtau_max)


def jfnk_matvec(X, q, R0, residual, shift, eps=FD_EPS):
    if not np.any(X):
        return np.zeros_like(X)
    return shift * X - (residual(q + eps * X) - R0) / eps


def _back_substitute(H, g):
    k = len(g)
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
    return y


def gmres_solve(matvec, b, kdim=30, max_restarts=10, rtol=1e-4, x0=None, precond=None, ortho="mgs"):
    """newton_krylov.py:79-151; ortho = "cgs2" restates the device option
    (classical Gram-Schmidt + one reorthogonalisation pass; not in the
    reference)."""
    n = len(b)
    bnorm = float(np.sqrt(b @ b))
    x = np.zeros(n) if x0 is None else x0.copy()
    if bnorm == 0.0:
        return x, 0, 0.0
    P = precond if precond is not None else (lambda v: v)
    total, relres = 0, np.inf
    for _ in range(max_restarts):
        r = b - matvec(x) if np.any(x) else b.copy()
        beta = float(np.sqrt(r @ r))
        relres = beta / bnorm
        if relres <= rtol:
            return x, total, relres
        m = kdim
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        j_done, breakdown = 0, False
        for j in range(m):
            w = matvec(P(V[j]))
            if not np.all(np.isfinite(w)):
                raise RuntimeError(f"non-finite Arnoldi vector at inner iteration {total + 1}")
            if ortho == "cgs2":
                h1 = V[:j + 1] @ w
                w = w - V[:j + 1].T @ h1
                h2 = V[:j + 1] @ w
                w = w - V[:j + 1].T @ h2
                H[:j + 1, j] = h1 + h2
            else:
                for i in range(j + 1):
                    H[i, j] = V[i] @ w
                    w = w - H[i, j] * V[i]
            H[j + 1, j] = float(np.sqrt(w @ w))
            total += 1
            if H[j + 1, j] > 1e-14 * bnorm:
                V[j + 1] = w / H[j + 1, j]
            else:
                breakdown = True
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            rho = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if rho == 0.0 else (H[j, j] / rho, H[j + 1, j] / rho)
            H[j, j], H[j + 1, j] = rho, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            j_done = j + 1
            relres = abs(g[j + 1]) / bnorm
            if relres <= rtol or breakdown:
                break
        y = _back_substitute(H[:j_done, :j_done], g[:j_done])
        x = x + P(V[:j_done].T @ y)
        if relres <= rtol or breakdown:
            return x, total, relres
    return x, total, relres


# ---------------------------------------------------------------------------
# element-Jacobi blocks

class Blocks:
    def __init__(self, disc: OracleDisc, shift, blocks, inv):
        self.disc, self.shift, self.blocks, self.inv = disc, shift, blocks, inv

    def apply(self, X):
        sz = self.disc.offsets[1]
        return np.einsum("mij,mj->mi", self.inv, X.reshape(-1, sz)).reshape(-1)


def element_block(disc: OracleDisc, e, q, frozen, eps=FD_EPS):
    sz = int(disc.offsets[1])
    n, nv = disc.n, disc.nv
    Q0 = q[e * sz:(e + 1) * sz]
    batch = np.repeat(Q0[None, :], sz + 1, axis=0)
    batch[np.arange(1, sz + 1), np.arange(sz)] += eps
    R = disc.element_residual(e, batch.reshape(sz + 1, n, n, nv), frozen).reshape(sz + 1, sz)
    return -(R[1:] - R[0]).T / eps


def assemble_blocks(disc: OracleDisc, q, shift, eps=FD_EPS):
    frozen = disc.freeze(q)
    M, sz = disc.mesh.n_elements, int(disc.offsets[1])
    B = np.empty((M, sz, sz))
    for e in range(M):
        B[e] = element_block(disc, e, q, frozen, eps)
        B[e][np.arange(sz), np.arange(sz)] += shift
    try:
        inv = np.linalg.inv(B)
    except np.linalg.LinAlgError:
        for e in range(M):
            c = np.linalg.cond(B[e])
            if not np.isfinite(c) or c > 1e15:
                raise RuntimeError(f"singular Jacobi block for element {e}")
        raise
    return Blocks(disc, shift, B, inv)


# ---------------------------------------------------------------------------
# block-sparse Jacobian and block ILU0 (newton_krylov.py:215-371)

def coupling_block(disc: OracleDisc, e, f, q, frozen, eps=FD_EPS):
    """-dR_e/dq_nb across face f of element e, by batched differencing of
    the neighbour state (newton_krylov.py:254-278)."""
    sz = int(disc.offsets[1])
    n, nv = disc.n, disc.nv
    nb = int(disc.nb[e, f])
    batch = np.repeat(q[nb * sz:(nb + 1) * sz][None, :], sz + 1, axis=0)
    batch[np.arange(1, sz + 1), np.arange(sz)] += eps
    q_rec, fvn_rec = disc.neighbor_record(e, f, batch.reshape(sz + 1, n, n, nv), frozen)
    Qe = np.broadcast_to(q[e * sz:(e + 1) * sz].reshape(n, n, nv), (sz + 1, n, n, nv))
    R = disc.element_residual(e, Qe, frozen, override=(f, q_rec, fvn_rec)).reshape(sz + 1, sz)
    return -(R[1:] - R[0]).T / eps


class SparseBlocks:
    """Block-CSR over element adjacency, columns sorted per row
    (SparseBlockMatrix, newton_krylov.py:218-251)."""

    def __init__(self, indptr, indices, blocks, sz):
        self.indptr, self.indices, self.blocks, self.sz = indptr, indices, blocks, sz
        self.n = len(indptr) - 1

    def entry(self, i, j):
        for k in range(self.indptr[i], self.indptr[i + 1]):
            if self.indices[k] == j:
                return k
        return -1

    def matvec(self, X):
        sz = self.sz
        out = np.zeros_like(X)
        for i in range(self.n):
            acc = np.zeros(sz)
            for k in range(self.indptr[i], self.indptr[i + 1]):
                j = int(self.indices[k])
                acc += self.blocks[k] @ X[j * sz:(j + 1) * sz]
            out[i * sz:(i + 1) * sz] = acc
        return out


def sparse_pattern(disc: OracleDisc):
    M = disc.mesh.n_elements
    indptr, indices = [0], []
    for i in range(M):
        cols = {i} | {int(disc.nb[i, f]) for f in range(4) if disc.interior[i, f]}
        indices.extend(sorted(cols))
        indptr.append(len(indices))
    return np.array(indptr), np.array(indices)


def assemble_sparse(disc: OracleDisc, q, shift, frozen=None, eps=FD_EPS):
    """A = shift I - dR/dq on the adjacency pattern: element blocks on the
    diagonal, coupling blocks accumulated per interior face in the mesh's
    face order (newton_krylov.py:281-311)."""
    frozen = disc.freeze(q) if frozen is None else frozen
    sz = int(disc.offsets[1])
    indptr, indices = sparse_pattern(disc)
    S = SparseBlocks(indptr, indices, [None] * len(indices), sz)
    for e in range(disc.mesh.n_elements):
        blk = element_block(disc, e, q, frozen, eps)
        blk[np.arange(sz), np.arange(sz)] += shift
        S.blocks[S.entry(e, e)] = blk
    for eL, fL, eR, fR, _ in disc.mesh.interior_faces:
        for e, f, nb in ((int(eL), int(fL), int(eR)), (int(eR), int(fR), int(eL))):
            k = S.entry(e, nb)
            blk = coupling_block(disc, e, f, q, frozen, eps)
            S.blocks[k] = blk if S.blocks[k] is None else S.blocks[k] + blk
    return S


class Ilu0:
    def __init__(self, F: SparseBlocks, diag_inv):
        self.F, self.diag_inv = F, diag_inv

    def apply(self, X):
        """LU y = X by block forward / backward sweeps (newton_krylov.py:348-368)."""
        F, sz = self.F, self.F.sz
        y = np.zeros_like(X)
        for i in range(F.n):
            acc = X[i * sz:(i + 1) * sz].copy()
            for k in range(F.indptr[i], F.indptr[i + 1]):
                j = int(F.indices[k])
                if j < i:
                    acc -= F.blocks[k] @ y[j * sz:(j + 1) * sz]
            y[i * sz:(i + 1) * sz] = acc
        out = np.zeros_like(X)
        for i in range(F.n - 1, -1, -1):
            acc = y[i * sz:(i + 1) * sz].copy()
            for k in range(F.indptr[i], F.indptr[i + 1]):
                j = int(F.indices[k])
                if j > i:
                    acc -= F.blocks[k] @ out[j * sz:(j + 1) * sz]
            out[i * sz:(i + 1) * sz] = self.diag_inv[i] @ acc
        return out


def ilu0_factor(A: SparseBlocks) -> Ilu0:
    """Block ILU with zero fill on A's pattern (newton_krylov.py:319-345)."""
    blocks = [b.copy() for b in A.blocks]
    F = SparseBlocks(A.indptr, A.indices, blocks, A.sz)
    diag_inv = [None] * F.n
    for i in range(F.n):
        row = list(range(F.indptr[i], F.indptr[i + 1]))
        for k in row:
            kk = int(F.indices[k])
            if kk >= i:
                continue
            blocks[k] = blocks[k] @ diag_inv[kk]
            krow = {int(F.indices[t]): t for t in range(F.indptr[kk], F.indptr[kk + 1])}
            for k2 in row:
                j = int(F.indices[k2])
                if j > kk and j in krow:
                    blocks[k2] = blocks[k2] - blocks[k] @ blocks[krow[j]]
        try:
            diag_inv[i] = np.linalg.inv(blocks[F.entry(i, i)])
        except np.linalg.LinAlgError:
            raise RuntimeError(f"singular ILU0 pivot block at element {i}")
    return Ilu0(F, diag_inv)


# ---------------------------------------------------------------------------
# pMG

RK_ALPHAS = (0.25, 1.0 / 3.0, 0.5, 1.0)
RK_CFL = 1.5


def rk_spectral_radius(disc: OracleDisc, q):
    """Per-element spectral-radius estimate lambda_e of dR/dq for the
    pseudo-transient RK smoother (NOT in the reference -- BASELINE.json's
    north star item (3); DESIGN.md section 4 "RK smoother"):

        h_e      = 4 |det J(0,0)| / max(L_xi, L_eta)   (L = centre-line lengths)
        lambda_e = A_p max_pts(|u| + c) / h_e + (p+1)^4 max_pts(nu) / h_e^2
        A_p      = 2 sqrt(2) rho_p, rho_p the spectral radius of the 1-D
                   upwind FR advection operator on [-1, 1] (Bloch analysis,
                   operators.fr_advection_radius)
        nu       = max(4/3 mu, kappa (gamma-1)) / rho   (NS), diffusivity (ADVD)
    """
    from paper_2202_09733_b200.mesh import pack_geometry
    g = pack_geometry(disc.mesh)
    a0, b0, c0, d0 = g[:, 0], g[:, 2], g[:, 4], g[:, 6]
    Lx = 2.0 * np.sqrt(a0 * a0 + b0 * b0)
    Ly = 2.0 * np.sqrt(c0 * c0 + d0 * d0)
    h = 4.0 * np.abs(a0 * d0 - c0 * b0) / np.maximum(Lx, Ly)
    M = disc.mesh.n_elements
    eqn = disc.eqn
    P = disc.p
    if eqn.kind == "advection-diffusion":
        ax, ay = eqn.advection
        a = np.full(M, np.sqrt(ax * ax + ay * ay))
        nu = np.full(M, float(eqn.diffusivity))
    else:
        Q = q.reshape(M, -1, 4)
        gam = eqn.gamma
        rho = Q[..., 0]
        u = Q[..., 1] / rho
        v = Q[..., 2] / rho
        p = (gam - 1.0) * (Q[..., 3] - 0.5 * rho * (u * u + v * v))
        a = (np.sqrt(u * u + v * v) + np.sqrt(gam * p / rho)).max(axis=1)
        if eqn.kind == "navier-stokes":
            nu = max(4.0 / 3.0 * eqn.mu, eqn.heat_conductivity * (gam - 1.0)) / rho.min(axis=1)
        else:
            nu = np.zeros(M)
    from paper_2202_09733_b200.operators import rk_adv_coef
    return rk_adv_coef(P) * a / h + float((P + 1) ** 4) * nu / (h * h)


class Level:
    def __init__(self, disc, nsweeps):
        self.disc, self.nsweeps = disc, nsweeps
        self.shift, self.q, self.S_base, self.S_extra, self.blocks = 0.0, None, 0.0, 0.0, None
        self.smoother, self.frozen_q, self.sparse, self.ilu = "ej", None, None, None
        self.lam = None  # RK smoother: per-element spectral radius at the frozen state

    def F(self, q):
        return self.shift * q - self.disc.residual(q)

    def defect(self):
        return (self.S_base - self.F(self.q)) + self.S_extra


def _transfer(T, data, n_in, n_out, nv):
    Q = data.reshape(-1, n_in, n_in, nv)
    return np.einsum("ai,bj,mijv->mabv", T, T, Q).reshape(-1)


class Pmg:
    """PmgContext (pmg.py:181-298): EJ and/or MBNK smoothers per level,
    optional switch to MBNK after ``switch_after`` solver cycles."""

    def __init__(self, disc: OracleDisc, levels, smooth=2, omega=1.0, smoother_shift=0.0, m_max=1,
                 smoother="ej", switch_after=None, mbnk_rtol=0.1, mbnk_maxiter=5,
                 rk_cfl=RK_CFL, rk_alphas=RK_ALPHAS):
        self.rk_cfl, self.rk_alphas = float(rk_cfl), tuple(float(a) for a in rk_alphas)
        degs = [int(t) for t in str(levels).split("-")]
        L = len(degs)

        def spread(text, cast):
            toks = [cast(t) for t in str(text).split("-")]
            return toks * L if len(toks) == 1 else toks
        sm, kinds = spread(smooth, int), spread(smoother, str)
        assert disc.p == degs[0] and len(sm) == L and len(kinds) == L
        self.omega, self.smoother_shift, self.m_max = omega, smoother_shift, m_max
        self.switch_after, self.mbnk_rtol, self.mbnk_maxiter = switch_after, mbnk_rtol, mbnk_maxiter
        self.levels = [Level(disc if k == 0 else OracleDisc(disc.mesh, p, disc.eqn), sm[k])
                       for k, p in enumerate(degs)]
        for lev, kind in zip(self.levels, kinds):
            lev.smoother = kind
        self.ops = [transfer_operators(degs[k], degs[k + 1]) for k in range(len(degs) - 1)]
        self.fallbacks = 0
        self.cycles_done = 0

    def _effective_smoother(self, k):
        if self.switch_after is not None and self.cycles_done >= self.switch_after:
            return "mbnk"
        return self.levels[k].smoother

    def _restrict(self, k, data):
        hi, lo = self.levels[k].disc, self.levels[k + 1].disc
        return _transfer(self.ops[k].gamma, data, hi.n, lo.n, hi.nv)

    def _prolong(self, k, data):
        hi, lo = self.levels[k].disc, self.levels[k + 1].disc
        return _transfer(self.ops[k].pi, data, lo.n, hi.n, hi.nv)

    def prepare(self, q, shift):
        self.q_outer = q.copy()
        self.R_outer = self.levels[0].disc.residual(q)
        self.shift = shift
        qk = q
        for k, lev in enumerate(self.levels):
            if k:
                qk = self._restrict(k - 1, qk)
            lev.shift = shift
            lev.frozen_q = qk.copy()
            if lev.smoother == "rk":   # matrix-free: no blocks on this level
                lev.blocks = None
                lev.lam = rk_spectral_radius(lev.disc, qk)
            else:
                lev.blocks = assemble_blocks(lev.disc, qk, shift + self.smoother_shift)
            lev.sparse = lev.ilu = None
        self.cycles_done = 0

    def _smooth(self, k):
        lev = self.levels[k]
        if lev.smoother == "rk" and self._effective_smoother(k) == "rk":
            # pseudo-transient explicit RK with local (per-element) pseudo-time
            # steps dtau_e = cfl / (s + lambda_e):  q <- q0 + alpha_j dtau_e d(q)
            npe = lev.disc.n * lev.disc.n * lev.disc.nv
            for _ in range(lev.nsweeps):
                q0 = lev.q
                dtau = self.rk_cfl / (lev.shift + lev.lam)
                for a in self.rk_alphas:
                    c = np.repeat(a * dtau, npe)
                    lev.q = q0 + c * lev.defect()
            return
        if self._effective_smoother(k) == "ej":
            for _ in range(lev.nsweeps):
                lev.q = lev.q + self.omega * lev.blocks.apply(lev.defect())
            return
        if lev.sparse is None:   # _ensure_sparse (pmg.py:239-243): the level's current shift
            lev.sparse = assemble_sparse(lev.disc, lev.frozen_q, lev.shift)
            lev.ilu = ilu0_factor(lev.sparse)
        for _ in range(lev.nsweeps):   # smooth_mbnk (pmg.py:167-175)
            r = lev.defect()
            dq, _, _ = gmres_solve(lev.sparse.matvec, r, kdim=self.mbnk_maxiter, max_restarts=1,
                                   rtol=self.mbnk_rtol, precond=lev.ilu.apply)
            lev.q = lev.q + dq

    def vcycle(self, k=0):
        lev = self.levels[k]
        self._smooth(k)
        if k == len(self.levels) - 1:
            return
        d = lev.defect()
        c = self.levels[k + 1]
        qb = self._restrict(k, lev.q)
        gd = self._restrict(k, d)
        c.q = qb.copy()
        c.S_base = c.F(qb)
        c.S_extra = gd
        self.vcycle(k + 1)
        lev.q = lev.q + self._prolong(k, c.q - qb)
        self._smooth(k)

    def precondition(self, X):
        fine = self.levels[0]
        fine.q = self.q_outer.copy()
        fine.S_base = self.shift * self.q_outer - self.R_outer
        fine.S_extra = X
        try:
            for _ in range(self.m_max):
                self.vcycle()
        except NonPhysicalStateError:
            self.fallbacks += 1
            if fine.blocks is None:   # RK fine level: the diagonal (shift) part of the EJ fallback
                return X * (1.0 / (self.shift + self.smoother_shift))
            return fine.blocks.apply(X)
        return fine.q - self.q_outer


def pmg_solve(ctx: Pmg, q0, dtau_init, dtau_max=1e12, max_iters=100, rtol=1e-4, shift0=0.0, const=0.0,
              refresh_every=0, ser=True):
    fine = ctx.levels[0]

    def outer_F(q):
        return shift0 * q - fine.disc.residual(q) - const

    q = q0.copy()
    Fk = outer_F(q)
    n0 = float(np.sqrt(Fk @ Fk))
    hist = [(n0, 1.0, dtau_init)]
    st = {"iters": 0, "vcycles": 0, "converged": True, "aborted": False, "history": hist, "final_norm": n0}
    if n0 == 0.0:
        return q, st
    dtau = dtau_init
    ctx.prepare(q, 1.0 / dtau + shift0)
    halved, k = False, 0
    while k < max_iters:
        s_tot = 1.0 / dtau + shift0
        for lev in ctx.levels:
            lev.shift = s_tot
        fine.q = q.copy()
        fine.S_base = 0.0
        fine.S_extra = q / dtau + const
        try:
            ctx.vcycle()
            qn = fine.q
            Fn = outer_F(qn)
        except NonPhysicalStateError:
            if halved:
                st["converged"], st["aborted"] = False, True
                return q, st
            halved, dtau = True, 0.5 * dtau
            continue
        k += 1
        ctx.cycles_done += 1
        st["iters"] = st["vcycles"] = k
        q, Fk = qn, Fn
        nk = float(np.sqrt(Fk @ Fk))
        if ser:
            dtau = ser_update(dtau, hist[-1][0], nk, dtau_max)
        hist.append((nk, nk / n0, dtau))
        st["final_norm"] = nk
        if nk / n0 <= rtol:
            return q, st
        if refresh_every and k % refresh_every == 0:
            ctx.prepare(q, 1.0 / dtau + shift0)
    st["converged"] = False
    return q, st


# ---------------------------------------------------------------------------
# PTC and steppers

def ptc_solve(F, q0, dtau_init, krylov, precond_factory=None, dtau_max=1e12, max_iters=100, rtol=1e-4,
              max_halvings=8, refresh_every=0, eps=FD_EPS, ser=True):
    q = q0.copy()
    Fk = F(q)
    n0 = float(np.sqrt(Fk @ Fk))
    st = {"iters": 0, "gmres_iters": 0, "converged": True, "aborted": False,
          "history": [(n0, 1.0, dtau_init)], "final_norm": n0, "gmres_per_iter": []}
    if n0 == 0.0:
        return q, st
    dtau = dtau_init
    P = precond_factory(q, dtau) if precond_factory else None
    halvings, k = 0, 0
    while k < max_iters:
        def matvec(X, q=q, Fk=Fk, dtau=dtau):
            if not np.any(X):
                return np.zeros_like(X)
            return X / dtau + (F(q + eps * X) - Fk) / eps
        try:
            dq, it, _ = gmres_solve(matvec, -Fk, precond=P, **krylov)
            st["gmres_iters"] += it
            st["gmres_per_iter"].append(it)
            qn = q + dq
            Fn = F(qn)
        except NonPhysicalStateError:
            halvings += 1
            if halvings > max_halvings:
                st["converged"], st["aborted"] = False, True
                return q, st
            dtau = 0.5 * dtau
            continue
        k += 1
        st["iters"] = k
        q, Fk = qn, Fn
        nk = float(np.sqrt(Fk @ Fk))
        if ser:
            dtau = ser_update(dtau, st["history"][-1][0], nk, dtau_max)
        st["history"].append((nk, nk / n0, dtau))
        st["final_norm"] = nk
        if nk / n0 <= rtol:
            return q, st
        if precond_factory and refresh_every and k % refresh_every == 0:
            P = precond_factory(q, dtau)
    st["converged"] = False
    return q, st


class Driver:
    """ImplicitDriver (harness.py:277-369) with a pMG or EJ preconditioner."""

    def __init__(self, disc: OracleDisc, precond="pmg", levels="3-2", smooth=2, smoother_shift=0.0,
                 kdim=30, max_restarts=10, gmres_rtol=1e-3, dtau_init=1e-3, ptc_rtol=1e-4,
                 max_iters=100, max_halvings=8, smoother="ej", rk_cfl=RK_CFL, rk_alphas=RK_ALPHAS, ortho="mgs"):
        self.disc, self.precond = disc, precond
        self.krylov = dict(kdim=kdim, max_restarts=max_restarts, rtol=gmres_rtol, ortho=ortho)
        self.ptc = dict(dtau_init=dtau_init, rtol=ptc_rtol, max_iters=max_iters, max_halvings=max_halvings)
        self.ctx = (Pmg(disc, levels, smooth, smoother_shift=smoother_shift, smoother=smoother, rk_cfl=rk_cfl,
                        rk_alphas=rk_alphas) if precond == "pmg" else None)
        self.records = []

    def _factory(self, shift0):
        if self.precond == "ej":
            def f(q, dtau):
                return assemble_blocks(self.disc, q, shift0 + 1.0 / dtau).apply
            return f

        def f(q, dtau):
            self.ctx.prepare(q, shift0 + 1.0 / dtau)
            return self.ctx.precondition
        return f

    def solve_stage(self, a_ii, dt, explicit, q0):
        adt = a_ii * dt

        def F(q):
            return (q - explicit) / adt - self.disc.residual(q)
        dtau = self.ptc["dtau_init"]
        q, st = ptc_solve(F, q0, dtau, self.krylov, self._factory(1.0 / adt),
                          rtol=self.ptc["rtol"], max_iters=self.ptc["max_iters"],
                          max_halvings=self.ptc["max_halvings"])
        self.records.append(("stage", st["iters"], st["gmres_iters"], st["gmres_per_iter"]))
        return q, st

    def esdirk_step(self, q, dt, a, b):
        s = len(b)
        R = [self.disc.residual(q)]
        qi = q
        for i in range(1, s):
            explicit = q + dt * sum(a[i, j] * R[j] for j in range(i))
            qi, st = self.solve_stage(a[i, i], dt, explicit, qi)
            if not st["converged"]:
                raise RuntimeError(f"stage {i + 1} nonlinear solve did not converge")
            R.append(self.disc.residual(qi))
        return q + dt * sum(b[j] * R[j] for j in range(s))

    def row_step(self, q, dt, a, cm, m, gamma):
        s = len(m)
        sigma = 1.0 / (gamma * dt)
        R_lin = self.disc.residual(q)
        if self.precond == "ej":
            P = assemble_blocks(self.disc, q, sigma).apply
        else:
            self.ctx.prepare(q, sigma)
            P = self.ctx.precondition
        K = []
        for i in range(s):
            y = q + sum(a[i, j] * K[j] for j in range(i)) if i else q
            rhs = self.disc.residual(y)
            for j in range(i):
                rhs = rhs + (cm[i, j] / dt) * K[j]
            Ki, it, rr = gmres_solve(lambda v: jfnk_matvec(v, q, R_lin, self.disc.residual, sigma), rhs,
                                     precond=P, **self.krylov)
            self.records.append(("row", 0, it, [it]))
            if not rr <= self.krylov["rtol"]:
                raise RuntimeError(f"stage {i + 1} linear solve did not converge")
            K.append(Ki)
        return q + sum(m[j] * K[j] for j in range(s))
