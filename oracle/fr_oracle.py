"""ORACLE (test infrastructure only -- never shipped, never measured as
the product).  A NumPy restatement of the reference pmgflow FR residual
and its element-local linearisation, used by tests/, by
``__graft_entry__.smoke()`` and by bench.py's cpu_baseline / reference
arm as the checker.  Pinned against golden vectors produced by running
the reference itself (tests/golden/make_golden.py).

Structure differs from the reference on purpose: instead of face
batches keyed by degree pairs (reference spatial.py:333-351) every
face value is gathered through the per-(element, face) link table that
the device kernels also consume, so the oracle doubles as a check of
that table.  Uniform polynomial degree only (the device path's scope).

Reference citations (``/root/reference/pkg/src/pmgflow/spatial.py``):
  primitive 94-100, euler_flux 103-110, roe_flux 113-163,
  viscous_flux_ns 166-180, boundary_state 183-203, _traces 398-405,
  _divergence 407-430, _transformed 432-437, _check_physical 439-446,
  _grad_vars 448-454, _one_sided_fvn 456-464, residual 501-570,
  _br1_gradient 594-603, _assemble 605-629, freeze 700-766,
  element_residual 768-853, neighbor_face_record 855-903,
  compute_forces 633-695.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2202_09733_b200.equation import EquationSpec, NonPhysicalStateError
from paper_2202_09733_b200.mesh import Mesh, element_geometry, face_links
from paper_2202_09733_b200.operators import face_operators

WALL_ADIABATIC, WALL_SLIP, FAR_FIELD, WALL_ISOTHERMAL = 0, 1, 2, 3


# ---------------------------------------------------------------------------
# pointwise physics (channel-last, any leading shape)

def primitive(q, gamma):
    rho = q[..., 0]
    u = q[..., 1] / rho
    v = q[..., 2] / rho
    p = (gamma - 1.0) * (q[..., 3] - 0.5 * rho * (u * u + v * v))
    return rho, u, v, p


def euler_flux(q, gamma):
    rho, u, v, p = primitive(q, gamma)
    mx, my, E = q[..., 1], q[..., 2], q[..., 3]
    fx = np.stack([mx, mx * u + p, mx * v, u * (E + p)], axis=-1)
    fy = np.stack([my, my * u, my * v + p, v * (E + p)], axis=-1)
    return fx, fy


def roe_flux(qL, qR, nrm, gamma):
    """Roe flux along unit normal, no entropy fix (spatial.py:113-163)."""
    nx, ny = nrm[..., 0], nrm[..., 1]
    rL, uL, vL, pL = primitive(qL, gamma)
    rR, uR, vR, pR = primitive(qR, gamma)
    HL = (qL[..., 3] + pL) / rL
    HR = (qR[..., 3] + pR) / rR
    sL, sR = np.sqrt(rL), np.sqrt(rR)
    w = sL / (sL + sR)
    u = w * uL + (1.0 - w) * uR
    v = w * vL + (1.0 - w) * vR
    H = w * HL + (1.0 - w) * HR
    c2 = (gamma - 1.0) * (H - 0.5 * (u * u + v * v))
    c = np.sqrt(c2)
    rb = sL * sR
    un = u * nx + v * ny
    du, dv = uR - uL, vR - vL
    dn = du * nx + dv * ny
    dt = -du * ny + dv * nx
    dp = pR - pL
    k1 = np.abs(un - c) * ((dp - rb * c * dn) / (2.0 * c2))
    k2 = np.abs(un) * ((rR - rL) - dp / c2)
    k3 = np.abs(un) * (rb * dt)
    k4 = np.abs(un + c) * ((dp + rb * c * dn) / (2.0 * c2))
    ut = -u * ny + v * nx
    diss = np.stack([
        k1 + k2 + k4,
        k1 * (u - c * nx) + k2 * u - k3 * ny + k4 * (u + c * nx),
        k1 * (v - c * ny) + k2 * v + k3 * nx + k4 * (v + c * ny),
        k1 * (H - c * un) + k2 * 0.5 * (u * u + v * v) + k3 * ut + k4 * (H + c * un),
    ], axis=-1)
    fxL, fyL = euler_flux(qL, gamma)
    fxR, fyR = euler_flux(qR, gamma)
    fn = 0.5 * (fxL + fxR) * nx[..., None] + 0.5 * (fyL + fyR) * ny[..., None]
    return fn - 0.5 * diss


def rusanov_flux(qL, qR, nrm, gamma):
    """Local Lax-Friedrichs flux along the unit normal (BASELINE configs'
    interface flux; not in the reference -- parity unpinned):
    F = 1/2 (f(qL) + f(qR)).n - 1/2 lambda (qR - qL),
    lambda = max(|u_L.n| + c_L, |u_R.n| + c_R)."""
    nx, ny = nrm[..., 0], nrm[..., 1]
    rL, uL, vL, pL = primitive(qL, gamma)
    rR, uR, vR, pR = primitive(qR, gamma)
    aL = np.abs(uL * nx + vL * ny) + np.sqrt(gamma * pL / rL)
    aR = np.abs(uR * nx + vR * ny) + np.sqrt(gamma * pR / rR)
    lam = np.maximum(aL, aR)
    fxL, fyL = euler_flux(qL, gamma)
    fxR, fyR = euler_flux(qR, gamma)
    fn = 0.5 * (fxL + fxR) * nx[..., None] + 0.5 * (fyL + fyR) * ny[..., None]
    return fn - (0.5 * lam)[..., None] * (qR - qL)


def viscous_flux(q, gx, gy, mu, kappa):
    """Stokes stress + Fourier heat flux from grads of (u, v, T)."""
    rho = q[..., 0]
    u, v = q[..., 1] / rho, q[..., 2] / rho
    ux, vx, Tx = gx[..., 0], gx[..., 1], gx[..., 2]
    uy, vy, Ty = gy[..., 0], gy[..., 1], gy[..., 2]
    d = ux + vy
    txx = mu * (2.0 * ux - (2.0 / 3.0) * d)
    tyy = mu * (2.0 * vy - (2.0 / 3.0) * d)
    txy = mu * (uy + vx)
    z = np.zeros_like(txx)
    fx = np.stack([z, txx, txy, u * txx + v * txy + kappa * Tx], axis=-1)
    fy = np.stack([z, txy, tyy, u * txy + v * tyy + kappa * Ty], axis=-1)
    return fx, fy


def ghost_state(q, tag, nrm, eqn: EquationSpec):
    """Outside state of a boundary face (spatial.py:183-203); tag codes."""
    if eqn.kind == "advection-diffusion":
        return np.zeros_like(q) if tag == FAR_FIELD else q.copy()
    if tag == FAR_FIELD:
        return np.broadcast_to(eqn.free_stream(), q.shape).copy()
    g = q.copy()
    if tag == WALL_SLIP:
        un = q[..., 1] * nrm[..., 0] + q[..., 2] * nrm[..., 1]
        g[..., 1] -= 2.0 * un * nrm[..., 0]
        g[..., 2] -= 2.0 * un * nrm[..., 1]
        return g
    g[..., 1] *= -1.0
    g[..., 2] *= -1.0
    return g


# ---------------------------------------------------------------------------

@dataclass
class Frozen:
    """Neighbour data held fixed for element-local linearisation
    (the content of the reference's freeze() records, spatial.py:750-765):
    q_nb: neighbour q trace aligned to this element's face points,
    fvn_nb: minus the neighbour's one-sided viscous normal flux, aligned."""

    q_nb: np.ndarray
    fvn_nb: np.ndarray | None


class OracleDisc:
    """FR residual on a uniform-degree quad mesh (CPU, NumPy)."""

    def __init__(self, mesh: Mesh, p: int, eqn: EquationSpec, dtype=np.float64):
        """``dtype=np.longdouble`` evaluates the same algorithm in x87
        extended precision (64-bit significand) on the float64 operators and
        geometry: the "truth" the full-size parity tests measure both the
        reference's and the device's float64 rounding against."""
        self.mesh, self.p, self.eqn = mesh, int(p), eqn
        self.dtype = dt = np.dtype(dtype)
        self.n = n = self.p + 1
        self.nv = eqn.nvars
        M = mesh.n_elements
        self.n_dofs = M * n * n * self.nv
        self.offsets = np.arange(M + 1) * (n * n * self.nv)
        self.degrees = np.full(M, self.p)
        self.D, self.eL, self.eR, self.lL, self.lR = (a.astype(dt) for a in face_operators(self.p))
        g = element_geometry(mesh, self.p)
        self.jac, self.det = g.jac.astype(dt), g.det.astype(dt)
        self.nrm, self.js = g.face_normals.astype(dt), g.face_jac.astype(dt)
        self.link, self.tag = face_links(mesh)
        self.interior = self.link[..., 0] >= 0
        k = np.arange(n)
        rev = self.link[..., 2].astype(bool)
        # own face point k meets neighbour face point kk
        self.kk = np.where(rev[..., None], n - 1 - k, k)
        self.nb = np.where(self.interior, self.link[..., 0], 0)
        self.fnb = np.where(self.interior, self.link[..., 1], 0)
        self.is_left = self.link[..., 3].astype(bool)

    # -- helpers -----------------------------------------------------------

    def _traces(self, Q):
        """(..., n, n, w) -> (..., 4, n, w), CCW face point order."""
        t0 = np.einsum("a,...abv->...bv", self.eL, Q)
        t1 = np.einsum("b,...abv->...av", self.eR, Q)
        t2 = np.einsum("a,...abv->...bv", self.eR, Q)[..., ::-1, :]
        t3 = np.einsum("b,...abv->...av", self.eL, Q)[..., ::-1, :]
        return np.stack([t0, t1, t2, t3], axis=-3)

    def _gather_nb(self, face_data):
        """Neighbour face data aligned to each element's own face points."""
        return face_data[self.nb[..., None], self.fnb[..., None], self.kk]

    def _div(self, e, Ft, Gt, Fc):
        """FR divergence for elements e (slice/array) -- spatial.py:407-430."""
        D, eL, eR, lL, lR = self.D, self.eL, self.eR, self.lL, self.lR
        js = self.js[e]
        div = (np.einsum("bc,...acv->...abv", D, Ft)
               + np.einsum("ac,...cbv->...abv", D, Gt))
        c1 = js[..., 1, None, None] * Fc[..., 1, :, :] - np.einsum("b,...abv->...av", eR, Ft)
        c3 = -js[..., 3, None, None] * Fc[..., 3, ::-1, :] - np.einsum("b,...abv->...av", eL, Ft)
        c2 = js[..., 2, None, None] * Fc[..., 2, ::-1, :] - np.einsum("a,...abv->...bv", eR, Gt)
        c0 = -js[..., 0, None, None] * Fc[..., 0, :, :] - np.einsum("a,...abv->...bv", eL, Gt)
        div = div + lR[None, :, None] * c1[..., :, None, :]
        div = div - lL[None, :, None] * c3[..., :, None, :]
        div = div + lR[:, None, None] * c2[..., None, :, :]
        div = div - lL[:, None, None] * c0[..., None, :, :]
        return div / self.det[e][..., None]

    def _grad_vars(self, Q):
        if self.eqn.kind == "advection-diffusion":
            return Q
        rho = Q[..., 0]
        p = primitive(Q, self.eqn.gamma)[3]
        return np.stack([Q[..., 1] / rho, Q[..., 2] / rho, p / rho], axis=-1)

    def _check(self, X, what):
        if self.eqn.kind == "advection-diffusion":
            return
        rho, _, _, p = primitive(X, self.eqn.gamma)
        bad = ~((rho > 0.0) & (p > 0.0))
        if bad.any():
            m = np.nonzero(bad.reshape(bad.shape[0], -1).any(axis=1))[0][0]
            raise NonPhysicalStateError(m, what)

    def _num_flux(self, qa, qc, nrm):
        if self.eqn.kind == "advection-diffusion":
            ax, ay = self.eqn.advection
            an = (ax * nrm[..., 0] + ay * nrm[..., 1])[..., None]
            return 0.5 * an * (qa + qc) - 0.5 * np.abs(an) * (qc - qa)
        if self.eqn.riemann == "rusanov":
            return rusanov_flux(qa, qc, nrm, self.eqn.gamma)
        return roe_flux(qa, qc, nrm, self.eqn.gamma)

    # -- viscous interface values: BR1 (reference) or LDG (option) ----------
    # LDG with C11 = 0 and the switch pointing from each interior face's L
    # element (is_left) to its R element: the common solution value is L's
    # trace, the common viscous flux R's one-sided flux.  Boundary faces keep
    # the BR1 treatment (ghost average, own one-sided flux).

    def _w_out(self, e, w_own, q_out):
        """Viscous variables of the outside state.  On "wall-isothermal"
        faces (BASELINE config 4; not in the reference) the ghost keeps the
        mirrored no-slip state of the inviscid flux but its temperature is
        2 T_w - T, so the BR1 common value holds T = T_w exactly."""
        w = self._grad_vars(q_out)
        if self.eqn.kind == "navier-stokes":
            iso = (self.tag[e] == WALL_ISOTHERMAL)[..., None]
            if np.any(iso):
                w = w.copy()
                w[..., 2] = np.where(iso, 2.0 * self.eqn.t_wall - w_own[..., 2], w[..., 2])
        return w

    def _common_w(self, inter, left_own, w_own, w_out):
        if self.eqn.viscous_scheme == "ldg":
            return np.where(inter, np.where(left_own, w_own, w_out), 0.5 * (w_own + w_out))
        return 0.5 * (w_own + w_out)

    def _common_fv(self, inter, left_own, fvn, fvn_nb):
        """fvn: own one-sided viscous normal flux; fvn_nb: MINUS the
        neighbour's (i.e. the neighbour's flux on our normal)."""
        if self.eqn.viscous_scheme == "ldg":
            return np.where(inter, np.where(left_own, fvn_nb, fvn), fvn)
        return np.where(inter, 0.5 * (fvn + fvn_nb), fvn)

    def _vflux(self, Q, gx, gy):
        if self.eqn.kind == "advection-diffusion":
            k = self.eqn.diffusivity
            return k * gx, k * gy
        return viscous_flux(Q, gx, gy, self.eqn.mu, self.eqn.heat_conductivity)

    def _gradient(self, e, W, What):
        """BR1 corrected gradients (spatial.py:594-603)."""
        J = self.jac[e]
        nx = self.nrm[e][..., 0][..., None, None]
        ny = self.nrm[e][..., 1][..., None, None]
        gx = self._div(e, J[..., 1, 1, None] * W, -J[..., 1, 0, None] * W, nx * What)
        gy = self._div(e, -J[..., 0, 1, None] * W, J[..., 0, 0, None] * W, ny * What)
        return gx, gy

    def _fvn(self, e, tr, gx, gy):
        fx, fy = self._vflux(tr, self._traces(gx), self._traces(gy))
        nrm = self.nrm[e][..., :, None, :]
        return fx * nrm[..., 0:1] + fy * nrm[..., 1:2]

    def _ghosts(self, e, tr):
        """Ghost states on every boundary face of elements e (others 0)."""
        gh = np.zeros_like(tr)
        tag = self.tag[e]
        for t in (WALL_ADIABATIC, WALL_SLIP, FAR_FIELD, WALL_ISOTHERMAL):
            sel = np.broadcast_to(tag == t, tr.shape[:-2])
            if sel.any():
                nrm = np.broadcast_to(self.nrm[e][..., None, :], tr.shape[:-1] + (2,))
                gh[sel] = ghost_state(tr[sel], t, nrm[sel], self.eqn)
        return gh

    def _assemble(self, e, Q, Fc, grads):
        if self.eqn.kind == "advection-diffusion":
            ax, ay = self.eqn.advection
            fx, fy = ax * Q, ay * Q
        else:
            fx, fy = euler_flux(Q, self.eqn.gamma)
        if grads is not None:
            fvx, fvy = self._vflux(Q, *grads)
            fx, fy = fx - fvx, fy - fvy
        J = self.jac[e]
        Ft = J[..., 1, 1, None] * fx - J[..., 0, 1, None] * fy
        Gt = -J[..., 1, 0, None] * fx + J[..., 0, 0, None] * fy
        return -self._div(e, Ft, Gt, Fc)

    # -- global residual (spatial.py:501-570) -------------------------------

    def residual(self, q):
        n, nv, eqn = self.n, self.nv, self.eqn
        e = slice(None)
        Q = np.asarray(q, dtype=self.dtype).reshape(-1, n, n, nv)
        self._check(Q, "state")
        tr = self._traces(Q)
        self._check(tr, "trace")
        inter = self.interior[..., None, None]
        gh = self._ghosts(e, tr)
        nb_tr = np.where(inter, self._gather_nb(tr), gh)
        # inviscid: evaluated on the L side's normal, -F to the R side
        left = (self.is_left | ~self.interior)[..., None, None]
        qa = np.where(left, tr, nb_tr)
        qc = np.where(left, nb_tr, tr)
        nrm_own = np.broadcast_to(self.nrm[:, :, None, :], tr.shape[:-1] + (2,))
        nrm_nb = self._gather_nb(nrm_own)
        nrm = np.where(left, nrm_own, nrm_nb)
        Fc = self._num_flux(qa, qc, nrm)
        Fc = np.where(left, Fc, -Fc)
        if not eqn.viscous:
            return self._assemble(e, Q, Fc, None).reshape(-1)
        W = self._grad_vars(Q)
        w_own = self._grad_vars(tr)
        lo = self.is_left[..., None, None]
        What = self._common_w(inter, lo, w_own, self._w_out(e, w_own, nb_tr))
        grads = self._gradient(e, W, What)
        fvn = self._fvn(e, tr, *grads)
        Fv = self._common_fv(inter, lo, fvn, -self._gather_nb(fvn))
        if eqn.kind == "navier-stokes":
            wall = (self.tag == WALL_ADIABATIC)[..., None]
            Fv[..., 3] = np.where(wall, 0.0, Fv[..., 3])
        return self._assemble(e, Q, Fc - Fv, grads).reshape(-1)

    # -- forces (spatial.py:633-695) ------------------------------------------

    def compute_forces(self, q):
        """(Fd, Fl, Cd, Cl): pressure p n minus the BR1 viscous traction
        tau n, integrated over the wall-tagged faces with the face weights
        and face_jac; coefficients with the reference length as area."""
        eqn = self.eqn
        if eqn.kind == "advection-diffusion":
            raise ValueError("forces are only defined for flow equations")
        wall = (self.tag == WALL_ADIABATIC) | (self.tag == WALL_SLIP) | (self.tag == WALL_ISOTHERMAL)
        if not wall.any():
            raise ValueError("mesh has no wall boundary faces")
        n, nv = self.n, self.nv
        Q = np.asarray(q, dtype=self.dtype).reshape(-1, n, n, nv)
        tr = self._traces(Q)
        grads = None
        if eqn.viscous:
            inter = self.interior[..., None, None]
            nb_tr = np.where(inter, self._gather_nb(tr), self._ghosts(slice(None), tr))
            w_own = self._grad_vars(tr)
            What = self._common_w(inter, self.is_left[..., None, None], w_own,
                                  self._w_out(slice(None), w_own, nb_tr))
            grads = self._gradient(slice(None), self._grad_vars(Q), What)
        from paper_2202_09733_b200.operators import gauss_rule
        wq = gauss_rule(n)[1]
        F = np.zeros(2)
        for e, f in np.argwhere(wall):
            t = tr[e, f]                                   # (n, 4)
            nrm = self.nrm[e, f]
            p = primitive(t, eqn.gamma)[3]
            contrib = p[:, None] * nrm[None, :]
            if grads is not None:
                gx_tr = self._traces(grads[0][e])[f]
                gy_tr = self._traces(grads[1][e])[f]
                ux, vx, uy, vy = gx_tr[:, 0], gx_tr[:, 1], gy_tr[:, 0], gy_tr[:, 1]
                div = ux + vy
                txx = eqn.mu * (2 * ux - (2.0 / 3.0) * div)
                tyy = eqn.mu * (2 * vy - (2.0 / 3.0) * div)
                txy = eqn.mu * (uy + vx)
                contrib = contrib - np.stack([txx * nrm[0] + txy * nrm[1], txy * nrm[0] + tyy * nrm[1]], axis=-1)
            F += np.einsum("k,kj->j", wq * self.js[e, f], contrib)
        qref = 0.5 * 1.0 * 1.0 ** 2 * eqn.ref_length
        return F[0], F[1], F[0] / qref, F[1] / qref

    # -- the same residual on all host cores (bench.py's reference arm) -------

    def _gather_nb_chunk(self, s, face_data):
        return face_data[self.nb[s][..., None], self.fnb[s][..., None], self.kk[s]]

    def _first_bad(self, X):
        if self.eqn.kind == "advection-diffusion":
            return -1
        rho, _, _, p = primitive(X, self.eqn.gamma)
        bad = ~((rho > 0.0) & (p > 0.0))
        rows = np.nonzero(bad.reshape(bad.shape[0], -1).any(axis=1))[0]
        return int(rows[0]) if rows.size else -1

    def residual_mt(self, q, threads=None, chunk=None):
        """``residual`` evaluated phase by phase over element chunks on a
        thread pool (NumPy releases the GIL inside its loops).  Every element
        sees exactly the operations of ``residual`` -- the result is bitwise
        identical (tests/test_oracle_golden.py) -- and a non-physical state
        raises the same error (state checks before trace checks, lowest
        element first)."""
        import concurrent.futures as cf
        import os
        T = int(threads or len(os.sched_getaffinity(0)))
        n, nv, eqn = self.n, self.nv, self.eqn
        Q = np.asarray(q, dtype=self.dtype).reshape(-1, n, n, nv)
        M = Q.shape[0]
        C = int(chunk or max(64, -(-M // (4 * T))))
        sl = [slice(a, min(a + C, M)) for a in range(0, M, C)]
        pool = getattr(self, "_pool", None)
        if pool is None or getattr(self, "_pool_threads", 0) != T:
            pool = self._pool = cf.ThreadPoolExecutor(T)
            self._pool_threads = T

        def run(fn):
            return list(pool.map(fn, sl))

        tr = np.empty((M, 4, n, nv), dtype=self.dtype)

        def p1(s):
            bs = self._first_bad(Q[s])
            tr[s] = self._traces(Q[s])
            bt = self._first_bad(tr[s])
            return (bs + s.start if bs >= 0 else -1, bt + s.start if bt >= 0 else -1)

        flags = run(p1)
        for k, what in ((0, "state"), (1, "trace")):
            hits = [f[k] for f in flags if f[k] >= 0]
            if hits:
                raise NonPhysicalStateError(min(hits), what)
        inter = self.interior[..., None, None]
        left = (self.is_left | ~self.interior)[..., None, None]
        nrm_nb = self.nrm[self.nb[..., None], self.fnb[..., None]]  # (M, 4, 1, 2)
        nb_tr = np.empty_like(tr)
        Fc = np.empty_like(tr)

        def p2(s):
            gh = self._ghosts(s, tr[s])
            nbt = np.where(inter[s], self._gather_nb_chunk(s, tr), gh)
            qa = np.where(left[s], tr[s], nbt)
            qc = np.where(left[s], nbt, tr[s])
            shp = tr[s].shape[:-1] + (2,)
            nrm_own = np.broadcast_to(self.nrm[s][:, :, None, :], shp)
            nrm = np.where(left[s], nrm_own, np.broadcast_to(nrm_nb[s], shp))
            F = self._num_flux(qa, qc, nrm)
            Fc[s] = np.where(left[s], F, -F)
            nb_tr[s] = nbt

        run(p2)
        R = np.empty_like(Q)
        if not eqn.viscous:
            def pe(s):
                R[s] = self._assemble(s, Q[s], Fc[s], None)
            run(pe)
            return R.reshape(-1)
        nw = self._grad_vars(Q[:1]).shape[-1]
        gx = np.empty((M, n, n, nw), dtype=self.dtype)
        gy = np.empty((M, n, n, nw), dtype=self.dtype)
        fvn = np.empty_like(tr)

        def p3(s):
            w_own = self._grad_vars(tr[s])
            What = self._common_w(inter[s], self.is_left[s][..., None, None], w_own,
                                  self._w_out(s, w_own, nb_tr[s]))
            gxs, gys = self._gradient(s, self._grad_vars(Q[s]), What)
            gx[s], gy[s] = gxs, gys
            fvn[s] = self._fvn(s, tr[s], gxs, gys)

        run(p3)

        def p4(s):
            Fv = self._common_fv(inter[s], self.is_left[s][..., None, None], fvn[s],
                                 -self._gather_nb_chunk(s, fvn))
            if eqn.kind == "navier-stokes":
                wall = (self.tag[s] == WALL_ADIABATIC)[..., None]
                Fv[..., 3] = np.where(wall, 0.0, Fv[..., 3])
            R[s] = self._assemble(s, Q[s], Fc[s] - Fv, (gx[s], gy[s]))

        run(p4)
        return R.reshape(-1)

    # -- frozen neighbour data (spatial.py:700-766) --------------------------

    def freeze(self, q) -> Frozen:
        n, nv = self.n, self.nv
        Q = np.asarray(q, dtype=self.dtype).reshape(-1, n, n, nv)
        tr = self._traces(Q)
        q_nb = self._gather_nb(tr)
        fvn_nb = None
        if self.eqn.viscous:
            inter = self.interior[..., None, None]
            gh = self._ghosts(slice(None), tr)
            nb_tr = np.where(inter, q_nb, gh)
            w_own = self._grad_vars(tr)
            What = self._common_w(inter, self.is_left[..., None, None], w_own,
                                  self._w_out(slice(None), w_own, nb_tr))
            fvn = self._fvn(slice(None), tr, *self._gradient(slice(None), self._grad_vars(Q), What))
            fvn_nb = -self._gather_nb(fvn)
        return Frozen(q_nb, fvn_nb)

    def element_residual(self, e: int, Q, frozen: Frozen, override=None):
        """Element-local residual with frozen neighbours, own-side fluxes
        throughout (spatial.py:768-853).  Q: (..., n, n, nv).  ``override``
        = (f, q_rec, fvn_rec) replaces face f's frozen record by batched
        records from ``neighbor_record`` (the reference's face_override,
        spatial.py:787-790)."""
        Q = np.asarray(Q, dtype=self.dtype)
        tr = self._traces(Q)
        inter = self.interior[e][:, None, None]
        q_nb = frozen.q_nb[e]
        fvn_nb = frozen.fvn_nb[e] if frozen.fvn_nb is not None else None
        if override is not None:
            f_ov, q_rec, fvn_rec = override
            q_nb = np.broadcast_to(q_nb, tr.shape).copy()
            q_nb[..., f_ov, :, :] = q_rec
            if fvn_nb is not None:
                fvn_nb = np.broadcast_to(fvn_nb, tr.shape).copy()
                fvn_nb[..., f_ov, :, :] = fvn_rec
        gh = self._ghosts(e, tr)
        q_out = np.where(inter, q_nb, gh)
        nrm = np.broadcast_to(self.nrm[e][:, None, :], tr.shape[:-1] + (2,))
        Fc = self._num_flux(tr, q_out, nrm)
        grads = None
        if self.eqn.viscous:
            lo = self.is_left[e][:, None, None]
            w_own = self._grad_vars(tr)
            What = self._common_w(inter, lo, w_own, self._w_out(e, w_own, q_out))
            grads = self._gradient(e, self._grad_vars(Q), What)
            fvn = self._fvn(e, tr, *grads)
            Fv = self._common_fv(inter, lo, fvn, fvn_nb)
            if self.eqn.kind == "navier-stokes":
                wall = (self.tag[e] == WALL_ADIABATIC)[:, None]
                Fv[..., 3] = np.where(wall, 0.0, Fv[..., 3])
            Fc = Fc - Fv
        return self._assemble(e, Q, Fc, grads)

    def neighbor_record(self, e: int, f: int, Q_nb, frozen: Frozen):
        """Face record of e's face f recomputed from a (batched) neighbour
        state Q_nb with the neighbour's own other faces frozen
        (spatial.py:855-903): the neighbour's trace and, when viscous, its
        one-sided viscous flux, aligned to e's face points, in the Frozen
        sign convention (fvn = -neighbour flux)."""
        nb, fnb, rev = int(self.nb[e, f]), int(self.fnb[e, f]), bool(self.link[e, f, 2])
        Q_nb = np.asarray(Q_nb, dtype=self.dtype)
        tr = self._traces(Q_nb)
        q_rec = tr[..., fnb, :, :]
        if rev:
            q_rec = q_rec[..., ::-1, :]
        fvn_rec = None
        if self.eqn.viscous:
            inter = self.interior[nb][:, None, None]
            gh = self._ghosts(nb, tr)
            q_out = np.where(inter, frozen.q_nb[nb], gh)
            w_own = self._grad_vars(tr)
            What = self._common_w(inter, self.is_left[nb][:, None, None], w_own,
                                  self._w_out(nb, w_own, q_out))
            gx, gy = self._gradient(nb, self._grad_vars(Q_nb), What)
            fv = self._fvn(nb, tr, gx, gy)[..., fnb, :, :]
            if rev:
                fv = fv[..., ::-1, :]
            fvn_rec = -fv
        return q_rec, fvn_rec

    # -- field helpers -------------------------------------------------------

    def free_stream_field(self):
        M = self.mesh.n_elements
        return np.broadcast_to(self.eqn.free_stream(),
                               (M, self.n, self.n, self.nv)).reshape(-1).copy()
