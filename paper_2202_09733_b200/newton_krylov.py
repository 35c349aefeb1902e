"""Device pseudo-transient Newton-Krylov -- drop-in for pmgflow.newton_krylov.

Control flow is the reference's, line for line
(``/root/reference/pkg/src/pmgflow/newton_krylov.py``); every vector
operation runs in libpmgflow_b200 on device-resident FP64 tensors:

* ``jfnk_matvec``        :71-76   fused prologue/epilogue R kernel
* ``gmres_solve``        :79-151  device MGS Arnoldi (deterministic
                                  reductions), host Givens / back-solve on
                                  the (m+1) x m Hessenberg matrix, one
                                  device->host sync per Arnoldi step
* ``assemble_element_blocks`` / ``BlockJacobian`` / ``ej_apply``
                         :157-214 FD blocks + batched Gauss-Jordan inverse
                                  + batched block GEMV
* ``ptc_solve`` / ``ser_update`` / ``PtcConfig`` / ``KrylovConfig``
                         :28-68, :377-437

Non-physical states are latched on the device and raised at the same
control-flow points the reference raises them (after the enqueued work
of a residual call is synchronised), so the PTC halving and pMG
fallback decisions are unchanged.  The MBNK smoother's block-sparse FD
Jacobian and block ILU0 (:220-371) are built here too
(``assemble_sparse_blocks``, ``ilu0_factor``, ``ilu0_apply``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, load
from .equation import NonPhysicalStateError
from .spatial import Discretization, raise_status
from .vec import active_partition, any_nonzero, dot, lincomb, nrm2, ptr, stream, to_device

FD_EPS = 1e-6


@dataclass
class PtcConfig:
    dtau_init: float = 1e-3
    dtau_max: float = 1e12
    max_iters: int = 100
    rtol: float = 1e-4
    atol: float | None = None
    ser: bool = True
    ser_as_printed: bool = False
    refresh_every: int = 0
    max_halvings: int = 1

    def __post_init__(self):
        if self.dtau_init <= 0:
            raise ValueError("dtau_init must be positive")


@dataclass
class KrylovConfig:
    """``ortho``: "mgs" -- modified Gram-Schmidt, the reference's order
    (newton_krylov.py:119-123), j + 2 all-reduces per Arnoldi step when the
    vectors are partitioned; "cgs2" -- classical Gram-Schmidt with one
    reorthogonalisation pass (an option, not in the reference): two
    multi-dots and the norm, 3 all-reduces per step whatever j, at the
    rounding of a different but equally stable orthogonalisation."""
    kdim: int = 30
    max_restarts: int = 10
    rtol: float = 1e-4
    ortho: str = "mgs"

    def __post_init__(self):
        if self.ortho not in ("mgs", "cgs2"):
            raise ValueError("gmres.ortho must be mgs or cgs2")
        if self.ortho == "cgs2" and self.kdim > 256:
            raise ValueError("gmres.ortho = cgs2 supports kdim <= 256")
        if self.kdim < 1:
            raise ValueError("kdim must be >= 1")
        # the device update x += P(V^T y) stages y in shared memory
        # (csrc/krylov_kernels.cu, GEMV_T_MAX_K); reject larger bases up front
        if self.kdim > 28991:
            raise ValueError("kdim must be <= 28991")


def ser_update(dtau, f_old, f_new, dtau_max, as_printed=False):
    """SER pseudo-step growth (newton_krylov.py:56-68)."""
    if f_old == 0.0 or f_new == 0.0:
        return dtau_max
    ratio = (f_new / f_old) if as_printed else (f_old / f_new)
    return min(dtau * ratio, dtau_max)


def _device_disc(residual):
    """The Discretization behind a bound ``disc.residual`` (fused path)."""
    d = getattr(residual, "__self__", None)
    if isinstance(d, Discretization) and getattr(residual, "__func__", None) is Discretization.residual:
        return d
    return None


def jfnk_matvec(X, q, R0, residual, shift, eps=FD_EPS, check_zero=True, sync=True):
    """(shift I - dR/dq) X ~ shift X - (R(q + eps X) - R0)/eps."""
    Xd = to_device(X)
    if check_zero and not any_nonzero(Xd):
        return torch.zeros_like(Xd)
    qd, R0d = to_device(q), to_device(R0)
    disc = _device_disc(residual)
    if disc is not None:
        out = disc.eval(qd, _lib.EPI_JV, X=Xd, eps=eps, s=shift, R0=R0d, check_status=sync)
    else:
        qp = lincomb((1.0, eps), (qd, Xd))
        Rp = to_device(residual(qp))
        out = lincomb((shift, -1.0 / eps, 1.0 / eps), (Xd, Rp, R0d))
    return out


def _back_substitute(H, g):
    k = len(g)
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
    return y


def _mgs_partitioned(V, j, w, thresh, Hd, flag):
    """Element-partitioned modified Gram-Schmidt over the
    rank's OWNED range of the strip vectors (halo entries are refreshed
    before anything reads them).  One rank: the fused pmgb_mgs on that
    range.  Several: pmgb_mgs_pass per projection with each partial dot
    all-reduced in-stream before the next pass applies it -- j+1 sequential
    all-reduces per Arnoldi step, the reference's MGS order
    (newton_krylov.py:119-127) -- then ||w|| from the all-reduced w . w.
    One host synchronisation per step (the Hessenberg column)."""
    lib = load()
    part = active_partition()
    n = V.shape[1]
    sz = n // part.n_local
    a0, n_o = part.owned.start * sz, (part.owned.stop - part.owned.start) * sz
    w_o = w[a0:a0 + n_o]
    row = lambda i: V.data_ptr() + (i * n + a0) * 8
    H = Hd[j]
    if part.world == 1:
        check(lib.pmgb_mgs(n_o, row(0), n, j, ptr(w_o), H.data_ptr(), thresh, flag.data_ptr(), stream()), "mgs")
    else:
        for i in range(j + 1):
            check(lib.pmgb_mgs_pass(n_o, ptr(w_o), row(i - 1) if i else None, H[i - 1:].data_ptr() if i else None,
                                    row(i), H[i:].data_ptr(), int(i == 0), flag.data_ptr() if i == 0 else None,
                                    stream()), "mgs_pass")
            part.allreduce_(H[i:i + 1], "sum")
            if i == 0:
                part.allreduce_(flag, "max")
        check(lib.pmgb_mgs_pass(n_o, ptr(w_o), row(j), H[j:].data_ptr(), ptr(w_o), H[j + 1:].data_ptr(), 0, None,
                                stream()), "mgs_pass")
        part.allreduce_(H[j + 1:j + 2], "sum")
        check(lib.pmgb_normalize_sqrt(n_o, ptr(w_o), H[j + 1:].data_ptr(), thresh, row(j + 1), stream()),
              "normalize_sqrt")
    hcol = H[:j + 2].cpu().numpy()
    return hcol, bool(int(flag.item()))


def _cgs2(V, j, w, thresh, Hd, flag, tmp):
    """Arnoldi step by classical Gram-Schmidt with reorthogonalisation
    (option gmres.ortho = cgs2): h1 = V w, w -= V^T h1, h2 = V w,
    w -= V^T h2, H[:j+1] = h1 + h2, H[j+1] = ||w||, V[j+1] = w / H[j+1] --
    over the rank's owned range when partitioned, each multi-dot and the
    norm all-reduced in-stream (3 all-reduces per step)."""
    lib = load()
    part = active_partition()
    n = V.shape[1]
    if part is None:
        a0, n_o = 0, n
    else:
        sz = n // part.n_local
        a0, n_o = part.owned.start * sz, (part.owned.stop - part.owned.start) * sz
    w_o = w[a0:a0 + n_o]
    base = V.data_ptr() + a0 * 8
    H = Hd[j]
    h1, h2 = H[:j + 1], tmp[:j + 1]
    flag.zero_()
    for k, h in enumerate((h1, h2)):
        check(lib.pmgb_multidot(n_o, base, n, j + 1, ptr(w_o), h.data_ptr(), flag.data_ptr() if k == 0 else None,
                                stream()), "multidot")
        if part is not None:
            part.allreduce_(h, "sum")
            if k == 0:
                part.allreduce_(flag, "max")
        check(lib.pmgb_gemv_sub(n_o, j + 1, base, n, h.data_ptr(), ptr(w_o), stream()), "gemv_sub")
    h1.add_(h2)
    check(lib.pmgb_dot(n_o, ptr(w_o), ptr(w_o), H[j + 1:].data_ptr(), stream()), "dot")
    if part is not None:
        part.allreduce_(H[j + 1:j + 2], "sum")
    check(lib.pmgb_normalize_sqrt(n_o, ptr(w_o), H[j + 1:].data_ptr(), thresh, base + (j + 1) * n * 8, stream()),
          "normalize_sqrt")
    hcol = H[:j + 2].cpu().numpy()
    return hcol, bool(int(flag.item()))


def gmres_solve(matvec, b, cfg: KrylovConfig, x0=None, precond=None):
    """Right-preconditioned restarted GMRES(m), newton_krylov.py:79-151.

    matvec / precond map device tensors to device tensors.  Returns
    (x, total inner iterations, final relative residual)."""
    lib = load()
    b = to_device(b)
    n = b.numel()
    bnorm = nrm2(b)
    x = torch.zeros_like(b) if x0 is None else to_device(x0).clone()
    if bnorm == 0.0:
        return x, 0, 0.0
    if precond is None:
        precond = lambda v: v
    m = cfg.kdim
    V = torch.empty((m + 1, n), dtype=torch.float64, device=b.device)
    Hd = torch.zeros((m, m + 2), dtype=torch.float64, device=b.device)
    flag = torch.zeros(1, dtype=torch.int32, device=b.device)
    tmp = torch.zeros(m + 1, dtype=torch.float64, device=b.device)
    thresh = 1e-14 * bnorm
    total = 0
    relres = np.inf
    for _ in range(cfg.max_restarts):
        if any_nonzero(x):
            r = lincomb((1.0, -1.0), (b, matvec(x)))
        else:
            r = b.clone()
        beta = nrm2(r)
        raise_status()
        relres = beta / bnorm
        if relres <= cfg.rtol:
            return x, total, relres
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        lincomb((1.0 / beta,), (r,), out=V[0])
        j_done = 0
        breakdown = False
        for j in range(m):
            w = matvec(precond(V[j]))
            if cfg.ortho == "cgs2":
                hcol, nonfinite = _cgs2(V, j, w, thresh, Hd, flag, tmp)
                raise_status()
            elif active_partition() is None:
                check(lib.pmgb_mgs(n, V.data_ptr(), n, j, ptr(w), Hd[j].data_ptr(), thresh,
                                   flag.data_ptr(), stream()), "mgs")
                hcol = Hd[j, :j + 2].cpu().numpy()
                raise_status()
                nonfinite = bool(int(flag.item()))
            else:
                hcol, nonfinite = _mgs_partitioned(V, j, w, thresh, Hd, flag)
                raise_status()
            if nonfinite:
                raise RuntimeError(f"non-finite Arnoldi vector at inner iteration {total + 1}")
            H[:j + 2, j] = hcol
            total += 1
            if not (H[j + 1, j] > thresh):
                breakdown = True
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            rho = np.hypot(H[j, j], H[j + 1, j])
            if rho == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j] = H[j, j] / rho
                sn[j] = H[j + 1, j] / rho
            H[j, j] = rho
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            j_done = j + 1
            relres = abs(g[j + 1]) / bnorm
            if relres <= cfg.rtol or breakdown:
                break
        y = _back_substitute(H[:j_done, :j_done], g[:j_done])
        yd = torch.as_tensor(y, device=b.device)
        comb = torch.empty_like(b)
        check(lib.pmgb_gemv_t(n, j_done, V.data_ptr(), n, yd.data_ptr(), comb.data_ptr(), stream()), "gemv_t")
        x = lincomb((1.0, 1.0), (x, to_device(precond(comb))))
        if relres <= cfg.rtol or breakdown:
            return x, total, relres
    return x, total, relres


# ---------------------------------------------------------------------------
# element-Jacobi blocks

class BlockJacobian:
    """Inverted diagonal blocks of (shift I - dR/dq), one per element.

    Device storage (include/pmgflow_b200.h): the in-place Gauss-Jordan
    factor ``XT`` (M, sz, sz) column-major and the pivot permutations
    ``perm`` (M, 2 sz) uint8, with B^-1[i][j] = X[p_i][q_j].  ``inv`` /
    ``blocks`` rebuild the reference's per-group (M, sz, sz) row-major
    arrays (newton_krylov.py:157-164) for inspection."""

    def __init__(self, disc: Discretization, shift: float, XT: torch.Tensor, perm: torch.Tensor, blocksT=None):
        self.disc = disc
        self.shift = shift
        self.XT = XT          # float64, or float32 with pmg.block_precision = fp32
        self.perm = perm
        self.blocksT = blocksT

    @property
    def precision(self) -> str:
        return "fp32" if self.XT.dtype == torch.float32 else "fp64"

    def demote(self) -> "BlockJacobian":
        """Store the factor in FP32 (round to nearest) and free the FP64
        copy; apply/update then read half the bytes (pmgb_blocks_demote)."""
        if self.XT.dtype == torch.float64:
            X32 = torch.empty(self.XT.shape, dtype=torch.float32, device=self.XT.device)
            check(load().pmgb_blocks_demote(self.XT.shape[0], self.XT.shape[1], self.XT.data_ptr(),
                                            X32.data_ptr(), stream()), "blocks_demote")
            self.XT = X32
        return self

    @property
    def inv(self):
        M, sz = self.XT.shape[0], self.XT.shape[1]
        X = self.XT.double().transpose(1, 2)
        p = self.perm[:, :sz].long()
        q = self.perm[:, sz:].long()
        rows = torch.gather(X, 1, p[:, :, None].expand(M, sz, sz))
        return [torch.gather(rows, 2, q[:, None, :].expand(M, sz, sz))]

    @property
    def blocks(self):
        if self.blocksT is None:
            raise AttributeError("blocks were not kept (keep_blocks=False)")
        return [self.blocksT.transpose(1, 2)]

    def apply(self, X):
        is_np = not isinstance(X, torch.Tensor)
        Xd = to_device(X, self.disc.device)
        out = torch.empty_like(Xd)
        fn = load().pmgb_ej_apply_f32 if self.XT.dtype == torch.float32 else load().pmgb_ej_apply
        check(fn(self.disc.mesh.n_elements, self.disc.elem_size, self.XT.data_ptr(),
                 self.perm.data_ptr(), ptr(Xd), ptr(out), stream()), "ej_apply")
        return out.cpu().numpy() if is_np else out

    def update(self, d: torch.Tensor, omega: float, base: torch.Tensor, out=None) -> torch.Tensor:
        """out = base + omega * B^-1 d (smooth_ej, pmg.py:164)."""
        if out is None:
            out = torch.empty_like(base)
        fn = load().pmgb_ej_update_f32 if self.XT.dtype == torch.float32 else load().pmgb_ej_update
        check(fn(self.disc.mesh.n_elements, self.disc.elem_size, self.XT.data_ptr(),
                 self.perm.data_ptr(), ptr(d), float(omega), ptr(base), ptr(out), stream()), "ej_update")
        return out


# ---------------------------------------------------------------------------
# block-sparse Jacobian (newton_krylov.py:215-311)

class _SparsePattern:
    """Element-adjacency block-CSR pattern (diagonal + face neighbours,
    columns sorted per row) and the coupling pairs in the reference's
    accumulation order, grouped into waves with distinct target slots
    (assemble_sparse_blocks, newton_krylov.py:281-311)."""

    def __init__(self, disc: Discretization):
        mesh = disc.mesh
        M = mesh.n_elements
        faces = np.asarray(mesh.interior_faces, dtype=np.int64).reshape(-1, 5)
        adj = [{i} for i in range(M)]
        for eL, fL, eR, fR, _ in faces.tolist():
            adj[eL].add(eR)
            adj[eR].add(eL)
        counts = np.array([len(a) for a in adj], dtype=np.int64)
        self.indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.indices = np.concatenate([sorted(a) for a in adj]).astype(np.int64) if M else np.zeros(0, np.int64)
        self.nnz = int(self.indptr[-1])
        rows = np.repeat(np.arange(M), counts)
        self.diag_slot = np.nonzero(self.indices == rows)[0]
        slot_of = {(int(r), int(c)): k for k, (r, c) in enumerate(zip(rows, self.indices))}
        pe, pf, ps, pa, pw = [], [], [], [], []
        contrib = np.zeros(self.nnz, dtype=np.int64)
        is_diag = self.indices == rows
        for eL, fL, eR, fR, _ in faces.tolist():
            for e, f, nb in ((eL, fL, eR), (eR, fR, eL)):
                k = slot_of[(e, nb)]
                pe.append(e)
                pf.append(f)
                ps.append(k)
                pa.append(1 if (is_diag[k] or contrib[k] > 0) else 0)
                pw.append(contrib[k])
                contrib[k] += 1
        order = np.argsort(np.asarray(pw, dtype=np.int64), kind="stable")
        self.pair_e = np.asarray(pe, dtype=np.int32)[order]
        self.pair_f = np.asarray(pf, dtype=np.int8)[order]
        self.pair_slot = np.asarray(ps, dtype=np.int32)[order]
        self.pair_add = np.asarray(pa, dtype=np.int8)[order]
        nw = int(max(pw) + 1) if pw else 0
        self.wave_ptr = np.concatenate([[0], np.cumsum(np.bincount(np.asarray(pw, dtype=np.int64),
                                                                    minlength=nw))]).astype(np.int64)
        # level schedules of the ILU0 sweeps: level(i) = 1 + max level of the
        # row's lower (upper) neighbours -- rows of one level are independent
        lo_lev = np.zeros(M, dtype=np.int64)
        for i in range(M):
            cols = self.indices[self.indptr[i]:self.indptr[i + 1]]
            low = cols[cols < i]
            lo_lev[i] = 1 + lo_lev[low].max() if low.size else 0
        up_lev = np.zeros(M, dtype=np.int64)
        for i in range(M - 1, -1, -1):
            cols = self.indices[self.indptr[i]:self.indptr[i + 1]]
            high = cols[cols > i]
            up_lev[i] = 1 + up_lev[high].max() if high.size else 0

        def schedule(lev):
            order = np.argsort(lev, kind="stable")
            ptr = np.concatenate([[0], np.cumsum(np.bincount(lev, minlength=int(lev.max()) + 1 if M else 0))])
            return order.astype(np.int32), ptr.astype(np.int64)
        self.lo_rows, self.lo_ptr = schedule(lo_lev)
        self.up_rows, self.up_ptr = schedule(up_lev)
        self.lo_diag = self.diag_slot[self.lo_rows].astype(np.int32)
        self.max_level_rows = int(max(np.diff(self.lo_ptr).max(), np.diff(self.up_ptr).max())) if M else 1
        # dense (slot, column) lists of each row's lower / upper blocks, CSR order
        ent = np.full((M, 2, 4, 2), -1, dtype=np.int32)
        for i in range(M):
            lo_n = up_n = 0
            for k in range(self.indptr[i], self.indptr[i + 1]):
                j = int(self.indices[k])
                if j < i:
                    if lo_n >= 4:
                        raise NotImplementedError("more than 4 lower block neighbours")
                    ent[i, 0, lo_n] = (k, j)
                    lo_n += 1
                elif j > i:
                    if up_n >= 4:
                        raise NotImplementedError("more than 4 upper block neighbours")
                    ent[i, 1, up_n] = (k, j)
                    up_n += 1
        self.row_entries = ent
        dev = disc.device
        self.d = {name: torch.as_tensor(np.ascontiguousarray(getattr(self, name)), device=dev)
                  for name in ("pair_e", "pair_f", "pair_slot", "pair_add", "lo_rows", "up_rows", "lo_diag")}
        self.d["diag_slot"] = torch.as_tensor(self.diag_slot.astype(np.int32), device=dev)
        self.d["indptr"] = torch.as_tensor(self.indptr.astype(np.int32), device=dev)
        self.d["indices"] = torch.as_tensor(self.indices.astype(np.int32), device=dev)
        self.d["lo_ptr"] = torch.as_tensor(self.lo_ptr.astype(np.int32), device=dev)
        self.d["up_ptr"] = torch.as_tensor(self.up_ptr.astype(np.int32), device=dev)
        self.d["barrier"] = torch.zeros(2, dtype=torch.int32, device=dev)
        self.d["row_entries"] = torch.as_tensor(self.row_entries, device=dev)

    def entry(self, i: int, j: int) -> int:
        lo, hi = int(self.indptr[i]), int(self.indptr[i + 1])
        k = lo + int(np.searchsorted(self.indices[lo:hi], j))
        return k if k < hi and self.indices[k] == j else -1


def sparse_pattern(disc: Discretization) -> _SparsePattern:
    pat = getattr(disc, "_sparse_pattern", None)
    if pat is None:
        pat = disc._sparse_pattern = _SparsePattern(disc)
    return pat


class SparseBlockMatrix:
    """Block-CSR over element adjacency (newton_krylov.py:218-251), on the
    device: ``blocksT`` (nnz, sz, sz) column-major (blocksT[k][c][r] =
    A_k[r][c]); ``indptr`` / ``indices`` as NumPy (host) with int32 device
    copies inside the pattern."""

    def __init__(self, disc: Discretization, pattern: _SparsePattern, blocksT: torch.Tensor):
        self.disc = disc
        self.pattern = pattern
        self.blocksT = blocksT
        self.n = disc.mesh.n_elements
        self.indptr = pattern.indptr
        self.indices = pattern.indices
        self.sizes = np.full(self.n, disc.elem_size, dtype=np.int64)

    @property
    def blocks(self):
        return self.blocksT.transpose(1, 2)

    def entry(self, i: int, j: int) -> int:
        return self.pattern.entry(i, j)

    def check_symmetric_pattern(self):
        for i in range(self.n):
            for k in range(self.indptr[i], self.indptr[i + 1]):
                j = int(self.indices[k])
                if self.entry(j, i) < 0:
                    raise ValueError(f"asymmetric sparsity: ({i},{j}) present, ({j},{i}) missing")

    def matvec(self, X, offsets=None):
        is_np = not isinstance(X, torch.Tensor)
        Xd = to_device(X, self.disc.device)
        out = torch.empty_like(Xd)
        pd = self.pattern.d
        check(load().pmgb_sparse_matvec(self.n, self.disc.elem_size, pd["indptr"].data_ptr(),
                                        pd["indices"].data_ptr(), self.blocksT.data_ptr(), ptr(Xd), ptr(out),
                                        stream()), "sparse_matvec")
        return out.cpu().numpy() if is_np else out


def assemble_sparse_blocks(disc: Discretization, data, shift: float, frozen=None,
                           eps: float = FD_EPS) -> SparseBlockMatrix:
    """A = shift I - dR/dq restricted to the element-adjacency pattern
    (newton_krylov.py:281-311): FD element blocks on the diagonal, FD
    coupling blocks through every interior face (neighbour face records
    recomputed from the perturbed neighbour, spatial.py:855-903),
    accumulated in the reference's face order."""
    del frozen  # the device freeze of ``data`` is recomputed (same values)
    q = to_device(data, disc.device)
    pat = sparse_pattern(disc)
    sz = disc.elem_size
    blocksT = torch.empty((pat.nnz, sz, sz), dtype=torch.float64, device=disc.device)
    d = pat.d
    wave_ptr = np.ascontiguousarray(pat.wave_ptr, dtype=np.int64)
    check(load().pmgb_sparse_assemble(disc._h, ptr(q), float(shift), float(eps), blocksT.data_ptr(),
                                      d["diag_slot"].data_ptr(), len(pat.pair_e), d["pair_e"].data_ptr(),
                                      d["pair_f"].data_ptr(), d["pair_slot"].data_ptr(), d["pair_add"].data_ptr(),
                                      wave_ptr.ctypes.data, len(wave_ptr) - 1, stream()), "sparse_assemble")
    return SparseBlockMatrix(disc, pat, blocksT)


class Ilu0Factors:
    """Block ILU0 factors on A's pattern (newton_krylov.py:314-316): ``F``
    the factored CSR values (column-major blocks), the pivot-block
    inverses as Gauss-Jordan factors (DX, DP)."""

    def __init__(self, pattern: SparseBlockMatrix, DX: torch.Tensor, DP: torch.Tensor):
        self.pattern = pattern
        self.DX = DX
        self.DP = DP

    @property
    def diag_inv(self):
        return BlockJacobian(self.pattern.disc, 0.0, self.DX, self.DP).inv[0]


def ilu0_factor(A: SparseBlockMatrix) -> Ilu0Factors:
    """Block ILU with zero fill on A's own pattern (newton_krylov.py:319-345),
    level-scheduled on the device.  Raises RuntimeError("singular ILU0 pivot
    block at element i")."""
    disc, pat = A.disc, A.pattern
    sz, M = disc.elem_size, A.n
    F = A.blocksT.clone()
    DX = torch.empty((M, sz, sz), dtype=torch.float64, device=disc.device)
    DP = torch.empty((M, 2 * sz), dtype=torch.uint8, device=disc.device)
    d = pat.d
    lp = np.ascontiguousarray(pat.lo_ptr, dtype=np.int64)
    check(load().pmgb_ilu0_factor(M, sz, d["indptr"].data_ptr(), d["indices"].data_ptr(), F.data_ptr(),
                                  DX.data_ptr(), DP.data_ptr(), len(lp) - 1, lp.ctypes.data,
                                  d["lo_rows"].data_ptr(), d["lo_diag"].data_ptr(), stream()), "ilu0_factor")
    raise_status()
    return Ilu0Factors(SparseBlockMatrix(disc, pat, F), DX, DP)


def ilu0_apply(fac: Ilu0Factors, X, offsets=None, fused: bool = True):
    """Solve LU y = X with the incomplete factors (newton_krylov.py:348-368):
    one cooperative launch walking the level schedule (``fused``), or one
    launch per level."""
    Fm = fac.pattern
    disc, pat = Fm.disc, Fm.pattern
    is_np = not isinstance(X, torch.Tensor)
    Xd = to_device(X, disc.device)
    y = torch.empty_like(Xd)
    out = torch.empty_like(Xd)
    d = pat.d
    nlo, nup = len(pat.lo_ptr) - 1, len(pat.up_ptr) - 1
    if fused:
        check(load().pmgb_ilu0_apply_fused(disc.elem_size, d["row_entries"].data_ptr(), Fm.blocksT.data_ptr(),
                                           fac.DX.data_ptr(), fac.DP.data_ptr(), nlo, d["lo_ptr"].data_ptr(), d["lo_rows"].data_ptr(), nup,
                                           d["up_ptr"].data_ptr(), d["up_rows"].data_ptr(), pat.max_level_rows,
                                           ptr(Xd), ptr(y), ptr(out), d["barrier"].data_ptr(), stream()),
              "ilu0_apply_fused")
    else:
        lp = np.ascontiguousarray(pat.lo_ptr, dtype=np.int64)
        up = np.ascontiguousarray(pat.up_ptr, dtype=np.int64)
        check(load().pmgb_ilu0_apply(Fm.n, disc.elem_size, d["indptr"].data_ptr(), d["indices"].data_ptr(),
                                     Fm.blocksT.data_ptr(), fac.DX.data_ptr(), fac.DP.data_ptr(), nlo,
                                     lp.ctypes.data, d["lo_rows"].data_ptr(), nup, up.ctypes.data,
                                     d["up_rows"].data_ptr(), ptr(Xd), ptr(y), ptr(out), stream()), "ilu0_apply")
    return out.cpu().numpy() if is_np else out


def assemble_element_blocks(disc: Discretization, data, shift: float, frozen=None, eps: float = FD_EPS,
                            keep_blocks: bool = True, precision: str = "fp64") -> BlockJacobian:
    """FD element blocks of shift I - dR/dq and their inverses.

    ``frozen`` is accepted for signature parity; the device freeze of
    ``data`` is always recomputed inside the assembly (same values).
    Raises RuntimeError("singular Jacobi block for element e")."""
    del frozen
    q = to_device(data, disc.device)
    M, sz = disc.mesh.n_elements, disc.elem_size
    XT = torch.empty((M, sz, sz), dtype=torch.float64, device=disc.device)
    perm = torch.empty((M, 2 * sz), dtype=torch.uint8, device=disc.device)
    blocksT = torch.empty_like(XT) if keep_blocks else XT
    disc.sync_halo(q)
    check(load().pmgb_blocks_assemble(disc._h, ptr(q), float(shift), float(eps), blocksT.data_ptr(),
                                      XT.data_ptr(), perm.data_ptr(), stream()), "blocks_assemble")
    raise_status()
    bj = BlockJacobian(disc, shift, XT, perm, blocksT if keep_blocks else None)
    if precision == "fp32":
        bj.demote()
    elif precision != "fp64":
        raise ValueError(f"unknown block precision {precision!r}")
    return bj


def ej_apply(blocks: BlockJacobian, X):
    return blocks.apply(X)


# ---------------------------------------------------------------------------
# pseudo-transient continuation (newton_krylov.py:377-437)

def _norm_checked(v: torch.Tensor) -> float:
    nv = nrm2(v)
    raise_status()
    return nv


def ptc_solve(F, q0, cfg: PtcConfig, krylov: KrylovConfig, precond_factory=None, eps: float = FD_EPS):
    """Drive F(q) = 0 by PTC with JFNK-GMRES; returns (q, stats).

    ``F`` maps device tensors to device tensors.  If it exposes
    ``fused_jv(X, q, Fk, dtau, eps)`` (the device stage function does),
    the PTC matvec X/dtau + (F(q+eps X) - Fk)/eps is one fused kernel
    chain; otherwise it is composed from F and device BLAS-1."""
    q = to_device(q0).clone()
    Fk = F(q)
    n0 = _norm_checked(Fk)
    stats = {"iters": 0, "gmres_iters": 0, "converged": True, "aborted": False,
             "history": [(n0, 1.0, cfg.dtau_init)], "final_norm": n0, "gmres_per_iter": []}
    if n0 == 0.0 or (cfg.atol is not None and n0 <= cfg.atol):
        return q, stats
    dtau = cfg.dtau_init
    P = precond_factory(q, dtau) if precond_factory else None
    fused = getattr(F, "fused_jv", None)
    halvings = 0
    k = 0
    while k < cfg.max_iters:
        # X = 0 returns 0 without evaluating F (newton_krylov.py:402-404)
        if fused is not None:
            def matvec(X, q=q, Fk=Fk, dtau=dtau):
                if not any_nonzero(X):
                    return torch.zeros_like(X)
                return fused(X, q, Fk, dtau, eps)
        else:
            def matvec(X, q=q, Fk=Fk, dtau=dtau):
                if not any_nonzero(X):
                    return torch.zeros_like(X)
                Fp = F(lincomb((1.0, eps), (q, X)))
                return lincomb((1.0 / dtau, 1.0 / eps, -1.0 / eps), (X, Fp, Fk))
        try:
            dq, it, _ = gmres_solve(matvec, lincomb((-1.0,), (Fk,)), krylov, precond=P)
            stats["gmres_iters"] += it
            stats["gmres_per_iter"].append(it)
            qn = lincomb((1.0, 1.0), (q, dq))
            Fn = F(qn)
            nk = _norm_checked(Fn)
        except NonPhysicalStateError:
            halvings += 1
            if halvings > cfg.max_halvings:
                stats["converged"] = False
                stats["aborted"] = True
                return q, stats
            dtau = 0.5 * dtau
            continue
        k += 1
        stats["iters"] = k
        q, Fk = qn, Fn
        if cfg.ser:
            prev = stats["history"][-1][0]
            dtau = ser_update(dtau, prev, nk, cfg.dtau_max, cfg.ser_as_printed)
        stats["history"].append((nk, nk / n0 if n0 else 0.0, dtau))
        stats["final_norm"] = nk
        if nk / n0 <= cfg.rtol or (cfg.atol is not None and nk <= cfg.atol):
            return q, stats
        if precond_factory and cfg.refresh_every and k % cfg.refresh_every == 0:
            P = precond_factory(q, dtau)
    stats["converged"] = False
    return q, stats
