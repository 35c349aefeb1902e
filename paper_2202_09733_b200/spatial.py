"""Device FR discretization -- the drop-in for pmgflow.spatial.Discretization.

Same constructor, attributes and entry points as the reference class
(``/root/reference/pkg/src/pmgflow/spatial.py:295-904``) for uniform
polynomial degree, with the arithmetic in libpmgflow_b200 (sm_100a FP64):

* ``residual(q)``           spatial.py:501-570 -> 3 kernels (traces,
                            one-sided viscous flux, common flux + FR
                            divergence); NonPhysicalStateError as the
                            reference (smallest element, state before trace)
* ``freeze(q)``             spatial.py:700-766 -> device traces + fvn
* ``element_residual``      spatial.py:768-853 -> one fused kernel
* ``free_stream_field/project/new_field`` (spatial.py:363-380)

Vectors may be NumPy arrays (copied in and out: the reference-facing
end-to-end path) or contiguous float64 CUDA tensors (device-resident
path used by the solvers).  A per-element degree map with more than one
degree constructs a ``MixedDiscretization`` (the reference's degree groups
with mortar faces, csrc/fr_mixed.cu): residual, freeze and
element_residual for Euler / Navier-Stokes with BR1.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, load
from .equation import KIND_CODE, EquationSpec, NonPhysicalStateError
from .mesh import TAG_CODE, Mesh, face_links, pack_geometry, solution_point_coords, element_geometry
from .operators import basis, face_operators, gauss_rule
from .vec import active_partition, ptr, require_cuda, stream, to_device

__all__ = ["Discretization", "SolutionField", "FrozenState", "NonPhysicalStateError",
           "EquationSpec", "raise_status"]


def raise_status(clear: bool = True):
    """Synchronise and turn the device status word into the reference's
    exceptions: NonPhysicalStateError(element, what) (spatial.py:27-32,
    439-446) or RuntimeError for a singular block (newton_krylov.py:207) or
    a singular ILU0 pivot block (newton_krylov.py:343)."""
    kind = ctypes.c_int32(0)
    elem = ctypes.c_int64(0)
    check(load().pmgb_status(stream(), ctypes.byref(kind), ctypes.byref(elem), int(clear)), "status")
    part = active_partition()
    if part is not None:
        # every rank raises the same exception: the smallest (kind, global
        # element) over the ranks (halo rows map to their owner's ids)
        k, e = part.reduce_status(kind.value, elem.value)
        kind.value, elem.value = k, e
    if kind.value == 1:
        raise NonPhysicalStateError(elem.value, "state")
    if kind.value == 2:
        raise NonPhysicalStateError(elem.value, "trace")
    if kind.value == 3:
        raise RuntimeError(f"singular Jacobi block for element {elem.value}")
    if kind.value == 4:
        raise RuntimeError(f"singular ILU0 pivot block at element {elem.value}")


def clear_status():
    check(load().pmgb_status_clear(stream()), "status_clear")


@dataclass
class SolutionField:
    nvars: int
    degrees: np.ndarray
    offsets: np.ndarray
    data: torch.Tensor

    @property
    def n_elements(self) -> int:
        return len(self.degrees)

    def element(self, e: int) -> torch.Tensor:
        n = int(self.degrees[e]) + 1
        return self.data[int(self.offsets[e]):int(self.offsets[e + 1])].view(n, n, self.nvars)

    def copy(self) -> "SolutionField":
        return SolutionField(self.nvars, self.degrees, self.offsets, self.data.clone())

    def with_data(self, data) -> "SolutionField":
        return SolutionField(self.nvars, self.degrees, self.offsets, data)


@dataclass
class FrozenState:
    """Device form of the reference's frozen records: every interior
    record (neighbour q trace, w trace, -fvn) is a gather from these."""

    qtr: torch.Tensor   # (M, 4, n, nv)
    fvn: torch.Tensor   # (M, 4, n, nv)


def _mesh_tables(mesh: Mesh):
    """Packed geometry records and face links depend on the mesh only (not
    on the degree): computed once per mesh object and reused by every pMG
    level and every Discretization built on it."""
    cache = getattr(mesh, "_pmgb_tables", None)
    if cache is None:
        links, tags = face_links(mesh)
        cache = (np.ascontiguousarray(pack_geometry(mesh)), links, tags)
        try:
            object.__setattr__(mesh, "_pmgb_tables", cache)
        except (AttributeError, TypeError):
            pass  # slotted / foreign mesh objects: no cache
    return cache


class Discretization:
    """FR residual operator on the device for a uniform-degree mesh (a
    mixed degree map yields a MixedDiscretization)."""

    def __new__(cls, mesh=None, degrees=None, eqn=None, device=None):
        if cls is Discretization and degrees is not None:
            d = np.asarray(degrees)
            if d.ndim == 1 and d.size and (d != d[0]).any():
                return super().__new__(MixedDiscretization)
        return super().__new__(cls)

    def __init__(self, mesh: Mesh, degrees, eqn: EquationSpec, device=None):
        require_cuda()
        self.mesh = mesh
        self.eqn = eqn
        degrees = np.asarray(degrees, dtype=np.int64)
        if degrees.ndim == 0:
            degrees = np.full(mesh.n_elements, int(degrees))
        if len(degrees) != mesh.n_elements:
            raise ValueError("degree map length does not match element count")
        if (degrees < 0).any():
            raise ValueError("degrees must be >= 0")
        if degrees.size and (degrees != degrees[0]).any():
            raise NotImplementedError("mixed-degree meshes are not on the device path yet")
        self.degrees = degrees
        self.p = int(degrees[0]) if degrees.size else 0
        if self.p > 5:
            raise NotImplementedError("device kernels cover p = 0..5")
        self.n = self.p + 1
        self.nvars = eqn.nvars
        self.elem_size = self.nvars * self.n * self.n
        M = mesh.n_elements
        self.offsets = np.arange(M + 1, dtype=np.int64) * self.elem_size
        self.n_dofs = int(self.offsets[-1])
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

        D, eL, eR, lL, lR = face_operators(self.p)
        self._ops = dict(D=np.ascontiguousarray(D), eL=eL.copy(), eR=eR.copy(), lL=lL.copy(),
                         lR=lR.copy(), xg=basis(self.p).points.copy())
        geom, links, tags = _mesh_tables(mesh)
        self._geom = geom
        self._links = np.ascontiguousarray(links)
        self._tags = np.ascontiguousarray(tags)
        self._qinf = np.ascontiguousarray(eqn.free_stream(), dtype=np.float64)
        dp = lambda a: a.ctypes.data_as(_lib.c_double_p)
        desc = _lib.DiscDesc(
            n_elem=M, degree=self.p, kind=KIND_CODE[eqn.kind],
            gamma=eqn.gamma, mu=eqn.mu, kappa=eqn.heat_conductivity if eqn.kind == "navier-stokes" else 0.0,
            adv_x=float(eqn.advection[0]), adv_y=float(eqn.advection[1]), diffusivity=eqn.diffusivity,
            free_stream=dp(self._qinf), D=dp(self._ops["D"]), eL=dp(self._ops["eL"]), eR=dp(self._ops["eR"]),
            lL=dp(self._ops["lL"]), lR=dp(self._ops["lR"]), xg=dp(self._ops["xg"]), geom=dp(self._geom),
            links=self._links.ctypes.data_as(_lib.c_int64_p), tags=self._tags.ctypes.data_as(_lib.c_int32_p),
            riemann=1 if eqn.riemann == "rusanov" else 0, viscous_scheme=1 if eqn.viscous_scheme == "ldg" else 0,
            wall_temperature=eqn.t_wall)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(load().pmgb_disc_create(ctypes.byref(desc), ctypes.byref(h)), "disc_create")
        self._h = h
        self._face_shape = (M, 4, self.n, self.nvars)
        self._geometry = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                load().pmgb_disc_destroy(h)
            except Exception:
                pass
            self._h = None

    def residual_path(self, want: str | None = None) -> str:
        """Residual kernel family in use: "rect" (axis-aligned rectangles,
        csrc/fr_rect.cu; chosen automatically when every element
        qualifies) or "general" (bilinear elements, csrc/fr_kernels.cu).
        ``want`` switches an eligible context (for A/B runs and tests);
        "rect2" / "rect4" pin the two- / four-kernel rectangle chain
        ("rect" takes the faster one per degree)."""
        code = {None: -1, "general": 0, "rect": 1, "rect4": 2, "rect2": 3}[want]
        r = load().pmgb_disc_residual_path(self._h, code)
        if r < 0:
            raise RuntimeError("residual_path: invalid context")
        return {0: "general", 1: "rect", 2: "rect4", 3: "rect2"}[r]

    # -- host-side conveniences ------------------------------------------------

    @property
    def geometry(self):
        if self._geometry is None:
            self._geometry = element_geometry(self.mesh, self.p)
        return self._geometry

    def new_field(self) -> SolutionField:
        return SolutionField(self.nvars, self.degrees, self.offsets,
                             torch.zeros(self.n_dofs, dtype=torch.float64, device=self.device))

    def free_stream_field(self) -> SolutionField:
        f = self.new_field()
        f.data.view(-1, self.nvars).copy_(torch.as_tensor(self.eqn.free_stream(), device=self.device))
        return f

    def project(self, fn) -> SolutionField:
        xy = solution_point_coords(self.mesh, self.p)
        vals = np.asarray(fn(xy[..., 0], xy[..., 1]), dtype=np.float64).reshape(-1)
        f = self.new_field()
        f.data.copy_(torch.as_tensor(vals))
        return f

    # -- forces (spatial.py:633-695) ---------------------------------------------

    def compute_forces(self, data):
        """Integrated wall force and coefficients (Fd, Fl, Cd, Cl): pressure
        plus BR1 viscous traction over all wall-tagged faces, computed on the
        device per wall face and summed here in face order; the coefficients
        use the reference length as the projected area."""
        eqn = self.eqn
        if eqn.kind == "advection-diffusion":
            raise ValueError("forces are only defined for flow equations")
        walls = getattr(self, "_wall_pairs", None)
        if walls is None:
            ef = np.argwhere((self._tags >= 0) & (self._tags != TAG_CODE["far-field"]))
            walls = self._wall_pairs = (
                len(ef),
                torch.as_tensor(ef[:, 0].astype(np.int32), device=self.device),
                torch.as_tensor(ef[:, 1].astype(np.int8), device=self.device))
        n_wall, we, wf = walls
        if n_wall == 0:
            raise ValueError("mesh has no wall boundary faces")
        q = to_device(data, self.device)
        out = torch.empty((n_wall, 2), dtype=torch.float64, device=self.device)
        w = np.ascontiguousarray(gauss_rule(self.n)[1], dtype=np.float64)
        check(load().pmgb_wall_forces(self._h, ptr(q), n_wall, we.data_ptr(), wf.data_ptr(),
                                      w.ctypes.data, out.data_ptr(), stream()), "wall_forces")
        F = out.cpu().numpy().sum(axis=0)
        qref = 0.5 * 1.0 * 1.0 ** 2 * eqn.ref_length  # rho_inf U_inf^2 A / 2
        return float(F[0]), float(F[1]), float(F[0] / qref), float(F[1] / qref)

    # -- device entry points ---------------------------------------------------

    def sync_halo(self, *vectors):
        """Refresh halo rows before a neighbour-reading kernel; a no-op on a
        whole mesh (partition.HaloDiscretization exchanges them)."""

    def coarsen(self, p: int) -> "Discretization":
        """The same mesh at degree p (pMG coarse levels, pmg.py:57-69)."""
        return Discretization(self.mesh, p, self.eqn, device=self.device)

    def eval(self, q: torch.Tensor, mode: int, out: torch.Tensor | None = None, *, X=None, eps=0.0,
             s=0.0, adt=0.0, dtau=0.0, R0=None, E=None, Sb=0.0, Se=0.0, Q0=None, dtau_e=None, alpha=0.0,
             check_status=False):
        """Fused residual + epilogue (see include/pmgflow_b200.h, PMGB_EPI_*)."""
        jv = X is not None and mode in (_lib.EPI_JV, _lib.EPI_STAGE_JV)
        self.sync_halo(q, X) if jv else self.sync_halo(q)
        if out is None:
            out = torch.empty(self.n_dofs, dtype=torch.float64, device=self.device)
        ep = _lib.Epilogue()
        ep.mode = mode
        ep.s, ep.eps, ep.adt, ep.dtau = float(s), float(eps), float(adt), float(dtau)
        ep.X = ptr(X) if X is not None else None
        ep.R0 = ptr(R0) if R0 is not None else None
        ep.E = ptr(E) if E is not None else None
        if isinstance(Sb, torch.Tensor):
            ep.Sb = ptr(Sb)
        else:
            ep.sb_scalar = float(Sb)
        if isinstance(Se, torch.Tensor):
            ep.Se = ptr(Se)
        else:
            ep.se_scalar = float(Se)
        ep.Q0 = ptr(Q0) if Q0 is not None else None
        ep.dtau_e = ptr(dtau_e) if dtau_e is not None else None
        ep.alpha = float(alpha)
        xp = ptr(X) if jv else None
        check(load().pmgb_eval(self._h, ptr(q), xp, float(eps), ctypes.byref(ep), ptr(out), stream()), "eval")
        if check_status:
            raise_status()
        return out

    def rk_lambda(self, q: torch.Tensor) -> torch.Tensor:
        """Per-element spectral-radius estimate for the RK smoother's local
        pseudo-time step (pmgb_rk_lambda; oracle: rk_spectral_radius)."""
        from .operators import rk_adv_coef
        lam = torch.empty(self.mesh.n_elements, dtype=torch.float64, device=self.device)
        check(load().pmgb_rk_lambda(self._h, ptr(q), rk_adv_coef(self.p), lam.data_ptr(), stream()), "rk_lambda")
        return lam

    def rk_dtau(self, lam: torch.Tensor, s: float, cfl: float) -> torch.Tensor:
        """Local pseudo-time steps cfl / (s + lam_e) (pmgb_rk_dtau)."""
        out = torch.empty_like(lam)
        check(load().pmgb_rk_dtau(lam.numel(), lam.data_ptr(), float(s), float(cfl), out.data_ptr(), stream()),
              "rk_dtau")
        return out

    def residual(self, data):
        """R(q); NumPy in -> NumPy out (end-to-end), CUDA tensor -> tensor."""
        if isinstance(data, torch.Tensor) and data.is_cuda:
            return self.eval(to_device(data), _lib.EPI_R, check_status=True)
        q = to_device(data, self.device)
        R = self.eval(q, _lib.EPI_R, check_status=True)
        return R.cpu().numpy()

    def residual_batch(self, qs, outs=None):
        """R(q) for a sequence of HOST arrays, copies overlapped with compute.

        Step i's host->device copy, step i-1's residual and step i-2's
        device->host copy run concurrently on three streams (two copy
        engines + compute), with double-buffered device staging.  Inputs
        should be pinned CPU tensors for full PCIe bandwidth; results go to
        ``outs`` (pinned CPU tensors, same length) or new pinned tensors.
        Raises NonPhysicalStateError after the batch if any step produced a
        non-physical state (the first one, as latched on the device)."""
        n = self.n_dofs
        qs = [q if isinstance(q, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(q)) for q in qs]
        if outs is None:
            outs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in qs]
        dev = self.device
        s_in, s_cmp, s_out = (torch.cuda.Stream(dev) for _ in range(3))
        dq = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
        dr = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in qs]
        ev_cmp = [torch.cuda.Event() for _ in qs]
        ev_out = [torch.cuda.Event() for _ in qs]
        cur = torch.cuda.current_stream(dev)
        for st in (s_in, s_cmp, s_out):
            st.wait_stream(cur)
        for i, q in enumerate(qs):
            b = i % 2
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(ev_cmp[i - 2])   # staging buffer free
                dq[b].copy_(q, non_blocking=True)
                ev_in[i].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[i])
                if i >= 2:
                    s_cmp.wait_event(ev_out[i - 2])  # result buffer drained
                self.eval(dq[b], _lib.EPI_R, dr[b])
                ev_cmp[i].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[i])
                outs[i].copy_(dr[b], non_blocking=True)
                ev_out[i].record(s_out)
        for st in (s_in, s_cmp, s_out):
            cur.wait_stream(st)
        raise_status()
        return outs

    def freeze(self, data) -> FrozenState:
        q = to_device(data, self.device)
        self.sync_halo(q)
        qtr = torch.empty(self._face_shape, dtype=torch.float64, device=self.device)
        fvn = torch.empty(self._face_shape, dtype=torch.float64, device=self.device)
        check(load().pmgb_freeze(self._h, ptr(q), qtr.data_ptr(), fvn.data_ptr(), stream()), "freeze")
        return FrozenState(qtr, fvn)

    def element_residual(self, e, Q, frozen: FrozenState):
        """Element-local residual with frozen neighbours; Q (..., n, n, nv).
        ``e`` may be an int or a per-instance array of element ids."""
        is_np = not isinstance(Q, torch.Tensor)
        Qd = to_device(Q, self.device)
        shape = Qd.shape
        Qf = Qd.reshape(-1, self.elem_size).contiguous()
        B = Qf.shape[0]
        el = torch.as_tensor(np.broadcast_to(np.asarray(e, dtype=np.int64), (B,)).copy(), device=self.device)
        out = torch.empty_like(Qf)
        check(load().pmgb_element_residual(self._h, el.data_ptr(), B, Qf.data_ptr(), frozen.qtr.data_ptr(),
                                           frozen.fvn.data_ptr(), out.data_ptr(), stream()), "element_residual")
        out = out.reshape(shape)
        return out.cpu().numpy() if is_np else out


@dataclass
class MixedFrozen:
    """Frozen neighbour records of a mixed-degree mesh at each element's own
    face points (spatial.py:700-766), padded to 6 points."""

    rq: torch.Tensor   # (M, 4, 6, 4) neighbour trace
    rw: torch.Tensor   # (M, 4, 6, 3) neighbour viscous variables
    rf: torch.Tensor   # (M, 4, 6, 4) minus the neighbour's one-sided viscous flux


class MixedDiscretization(Discretization):
    """Device FR discretization with a per-element degree map (p = 0..5):
    the reference's degree groups and mortar faces (spatial.py:295-359,
    468-585) on csrc/fr_mixed.cu.  Euler / Navier-Stokes, Roe or Rusanov,
    BR1 (the reference's only viscous scheme); flat vectors in the
    reference's layout (element e at offsets[e])."""

    def __init__(self, mesh: Mesh, degrees, eqn: EquationSpec, device=None):
        from .operators import mixed_tables
        require_cuda()
        self.mesh, self.eqn = mesh, eqn
        degrees = np.asarray(degrees, dtype=np.int64)
        if len(degrees) != mesh.n_elements:
            raise ValueError("degree map length does not match element count")
        if (degrees < 0).any():
            raise ValueError("degrees must be >= 0")
        if degrees.max() > 5:
            raise NotImplementedError("device kernels cover p = 0..5")
        if eqn.kind not in ("euler", "navier-stokes"):
            raise NotImplementedError("mixed-degree device path: Euler / Navier-Stokes")
        if eqn.viscous_scheme != "br1":
            raise NotImplementedError("mixed-degree device path: BR1 viscous fluxes (the reference's scheme)")
        self.degrees = degrees
        self.p = int(degrees.max())
        self.nvars = eqn.nvars
        sizes = self.nvars * (degrees + 1) ** 2
        self.offsets = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
        self.n_dofs = int(self.offsets[-1])
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        geom, links, tags = _mesh_tables(mesh)
        self._geom, self._links, self._tags = geom, np.ascontiguousarray(links), np.ascontiguousarray(tags)
        self._qinf = np.ascontiguousarray(eqn.free_stream(), dtype=np.float64)
        self._ops, self._xfer = mixed_tables()
        self._deg32 = np.ascontiguousarray(degrees, dtype=np.int32)
        z = np.zeros(36)
        dp = lambda a: a.ctypes.data_as(_lib.c_double_p)  # noqa: E731
        desc = _lib.DiscDesc(
            n_elem=mesh.n_elements, degree=0, kind=KIND_CODE[eqn.kind], gamma=eqn.gamma, mu=eqn.mu,
            kappa=eqn.heat_conductivity if eqn.kind == "navier-stokes" else 0.0, adv_x=0.0, adv_y=0.0,
            diffusivity=0.0, free_stream=dp(self._qinf), D=dp(z), eL=dp(z), eR=dp(z), lL=dp(z), lR=dp(z),
            xg=dp(z), geom=dp(self._geom), links=self._links.ctypes.data_as(_lib.c_int64_p),
            tags=self._tags.ctypes.data_as(_lib.c_int32_p), riemann=1 if eqn.riemann == "rusanov" else 0,
            viscous_scheme=0, wall_temperature=eqn.t_wall)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(load().pmgb_mdisc_create(ctypes.byref(desc), self._deg32.ctypes.data_as(_lib.c_int32_p),
                                           dp(self._ops), dp(self._xfer), ctypes.byref(h)), "mdisc_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                load().pmgb_mdisc_destroy(h)
            except Exception:
                pass
            self._h = None

    def residual_path(self, want=None) -> str:
        return "mixed"

    def coarsen(self, p):
        raise NotImplementedError("mixed-degree pMG levels: build the nested degree maps with "
                                  "p_adapt.nest_hierarchy and construct each level directly")

    def eval(self, q, mode: int, out=None, *, X=None, eps=0.0, s=0.0, adt=0.0, dtau=0.0, R0=None, E=None,
             Sb=0.0, Se=0.0, Q0=None, dtau_e=None, alpha=0.0, check_status=False):
        if mode == _lib.EPI_RK:
            raise NotImplementedError("the RK smoother epilogue is uniform-degree only")
        if out is None:
            out = torch.empty(self.n_dofs, dtype=torch.float64, device=self.device)
        ep = _lib.Epilogue()
        ep.mode = mode
        ep.s, ep.eps, ep.adt, ep.dtau = float(s), float(eps), float(adt), float(dtau)
        ep.X = ptr(X) if X is not None else None
        ep.R0 = ptr(R0) if R0 is not None else None
        ep.E = ptr(E) if E is not None else None
        if isinstance(Sb, torch.Tensor):
            ep.Sb = ptr(Sb)
        else:
            ep.sb_scalar = float(Sb)
        if isinstance(Se, torch.Tensor):
            ep.Se = ptr(Se)
        else:
            ep.se_scalar = float(Se)
        jv = X is not None and mode in (_lib.EPI_JV, _lib.EPI_STAGE_JV)
        check(load().pmgb_mdisc_eval(self._h, ptr(q), ptr(X) if jv else None, float(eps), ctypes.byref(ep),
                                     ptr(out), stream()), "mdisc_eval")
        if check_status:
            raise_status()
        return out

    def freeze(self, data) -> MixedFrozen:
        q = to_device(data, self.device)
        M = self.mesh.n_elements
        rq = torch.zeros((M, 4, 6, 4), dtype=torch.float64, device=self.device)
        rw = torch.zeros((M, 4, 6, 3), dtype=torch.float64, device=self.device)
        rf = torch.zeros((M, 4, 6, 4), dtype=torch.float64, device=self.device)
        check(load().pmgb_mdisc_freeze(self._h, ptr(q), rq.data_ptr(), rw.data_ptr(), rf.data_ptr(), stream()),
              "mdisc_freeze")
        return MixedFrozen(rq, rw, rf)

    def element_residual(self, e, Q, frozen: MixedFrozen):
        """Element-local residual (spatial.py:768-853); ``e`` an int or an
        array of elements of one degree, Q (..., n, n, nv)."""
        is_np = not isinstance(Q, torch.Tensor)
        els = np.atleast_1d(np.asarray(e, dtype=np.int64))
        p = int(self.degrees[els[0]])
        if (self.degrees[els] != p).any():
            raise ValueError("element_residual: the elements must share one degree")
        n = p + 1
        Qd = to_device(Q, self.device)
        shape = Qd.shape
        Qf = Qd.reshape(-1, self.nvars * n * n).contiguous()
        B = Qf.shape[0]
        el = torch.as_tensor(np.broadcast_to(els, (B,)).copy() if els.size == 1 else els, device=self.device)
        out = torch.empty_like(Qf)
        check(load().pmgb_mdisc_element_residual(self._h, p, el.data_ptr(), B, Qf.data_ptr(), frozen.rq.data_ptr(),
                                                 frozen.rw.data_ptr(), frozen.rf.data_ptr(), out.data_ptr(),
                                                 stream()), "mdisc_element_residual")
        out = out.reshape(shape)
        return out.cpu().numpy() if is_np else out
