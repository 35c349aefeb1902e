"""Device polynomial multigrid -- drop-in for pmgflow.pmg.

Control flow follows the reference (``/root/reference/pkg/src/pmgflow/pmg.py``)
line for line; vectors live on the device:

* ``PHierarchy`` / ``PmgPrecondConfig``          :29-86 (host, identical)
* ``_restrict`` / ``_prolong``                   :117-136 -> pmgb_transfer
* ``LevelState.F`` / ``defect``                  :142-159 -> fused R epilogues
* ``smooth_ej``                                  :162-164 -> defect kernel chain +
                                                 fused block-GEMV update
* ``smooth_mbnk``                                :167-175 -> GMRES on the device
                                                 block-sparse Jacobian + block ILU0
* ``smooth_rk`` (no reference counterpart; BASELINE north star item 3):
  matrix-free pseudo-transient explicit RK with local pseudo-time steps,
  one fused residual epilogue per stage (PMGB_EPI_RK) -- no element blocks
  on that level, which is what lets config 5's p=5 fine level fit
* ``PmgContext.prepare/vcycle/precondition``     :181-298 (incl. switch_after,
                                                 _ensure_sparse :213-253)
* ``pmg_solve``                                  :308-374

Uniform-degree levels only (mixed degrees: SURVEY 8(f) rank 3).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import newton_krylov as nk
from ._lib import check, load
from .equation import NonPhysicalStateError
from .operators import transfer_operators
from .spatial import Discretization, raise_status
from .vec import active_partition, lincomb, nrm2, ptr, stream, to_device


@dataclass(frozen=True)
class PHierarchy:
    levels: tuple
    smooth: tuple
    smoothers: tuple
    switch_after: int | None = None

    def __post_init__(self):
        if any(b >= a for a, b in zip(self.levels, self.levels[1:])):
            raise ValueError("level degrees must be strictly decreasing")
        if len(self.smooth) != len(self.levels) or len(self.smoothers) != len(self.levels):
            raise ValueError("per-level settings must match the level count")
        if any(n < 1 for n in self.smooth):
            raise ValueError("smoothing counts must be positive")
        if any(s not in ("ej", "mbnk", "rk") for s in self.smoothers):
            raise ValueError("smoother kinds are 'ej', 'mbnk' or 'rk'")

    @classmethod
    def parse(cls, levels: str, smooth: str = "2", smoother: str = "ej", switch_after=None):
        degs = tuple(int(t) for t in str(levels).split("-"))
        L = len(degs)

        def spread(text, cast):
            toks = [cast(t) for t in str(text).split("-")]
            if len(toks) == 1:
                toks = toks * L
            if len(toks) != L:
                raise ValueError(f"{text!r} does not match {L} hierarchy levels")
            return tuple(toks)

        return cls(degs, spread(smooth, int), spread(smoother, str), switch_after)

    def label(self) -> str:
        return "p{" + "-".join(str(p) for p in self.levels) + "}"


@dataclass
class PmgPrecondConfig:
    hierarchy: PHierarchy
    m_max: int = 1
    mbnk_rtol: float = 0.1
    mbnk_maxiter: int = 5
    omega: float = 1.0
    smoother_shift: float = 0.0
    rk_cfl: float = 1.5
    rk_alphas: tuple = (0.25, 1.0 / 3.0, 0.5, 1.0)
    # storage of the EJ block factors: fp64 (reference) or fp32 (option:
    # FP32 storage, FP64 arithmetic -- halves the EJ apply's HBM bytes)
    block_precision: str = "fp64"
    # precondition() as a CUDA-graph replay of its V-cycles: "auto" (meshes up
    # to PmgContext.GRAPH_AUTO_DOFS unknowns, where the cycle is launch-bound), "on", "off"
    graph: str = "auto"

    def __post_init__(self):
        if self.block_precision not in ("fp64", "fp32"):
            raise ValueError(f"unknown block precision {self.block_precision!r}")
        if self.graph not in ("auto", "on", "off"):
            raise ValueError(f"unknown graph mode {self.graph!r}")
        if self.m_max < 1:
            raise ValueError("m_max must be >= 1")
        if self.rk_cfl <= 0.0 or not self.rk_alphas:
            raise ValueError("RK smoother needs rk_cfl > 0 and at least one stage")


class _Transfer:
    """Gamma / Pi between two uniform-degree levels (pmg.py:92-114)."""

    def __init__(self, hi: Discretization, lo: Discretization):
        self.hi, self.lo = hi, lo
        self.M = hi.mesh.n_elements
        self.nv = hi.nvars
        self.nh, self.nl = hi.n, lo.n
        ops = transfer_operators(hi.p, lo.p)
        self.gamma = np.ascontiguousarray(ops.gamma, dtype=np.float64)
        self.pi = np.ascontiguousarray(ops.pi, dtype=np.float64)

    def restrict(self, src: torch.Tensor, out=None) -> torch.Tensor:
        if out is None:
            out = torch.empty(self.lo.n_dofs, dtype=torch.float64, device=src.device)
        check(load().pmgb_transfer(self.M, self.nv, self.nh, self.nl,
                                   self.gamma.ctypes.data_as(_lib.c_double_p), ptr(src), None, ptr(out), 0,
                                   stream()), "restrict")
        return out

    def prolong_add(self, lo: torch.Tensor, lo_base: torch.Tensor, hi: torch.Tensor) -> torch.Tensor:
        """hi += (Pi (x) Pi)(lo - lo_base), in place."""
        check(load().pmgb_transfer(self.M, self.nv, self.nl, self.nh,
                                   self.pi.ctypes.data_as(_lib.c_double_p), ptr(lo), ptr(lo_base), ptr(hi), 1,
                                   stream()), "prolong")
        return hi

    def prolong(self, lo: torch.Tensor) -> torch.Tensor:
        out = torch.empty(self.hi.n_dofs, dtype=torch.float64, device=lo.device)
        check(load().pmgb_transfer(self.M, self.nv, self.nl, self.nh,
                                   self.pi.ctypes.data_as(_lib.c_double_p), ptr(lo), None, ptr(out), 0,
                                   stream()), "prolong")
        return out


class LevelState:
    """One pMG level: F(q) = s q - R(q) = S with S = S_base + S_extra."""

    def __init__(self, disc: Discretization, shift: float = 0.0, q=None, S_base=0.0, S_extra=0.0,
                 nsweeps: int = 1, smoother: str = "ej", blocks=None):
        self.disc = disc
        self.shift = shift
        self.q = None if q is None else to_device(q, disc.device)
        self.S_base = S_base if not isinstance(S_base, np.ndarray) else to_device(S_base, disc.device)
        self.S_extra = S_extra if not isinstance(S_extra, np.ndarray) else to_device(S_extra, disc.device)
        self.nsweeps = nsweeps
        self.smoother = smoother
        self.blocks = blocks
        self.frozen_q = None
        self.sparse = None  # SparseBlockMatrix (MBNK)
        self.ilu = None     # Ilu0Factors (MBNK)
        self.lam = None     # per-element spectral radius at the frozen state (RK)

    def F(self, q) -> torch.Tensor:
        return self.disc.eval(to_device(q, self.disc.device), _lib.EPI_F, s=self.shift)

    def defect(self) -> torch.Tensor:
        return self.disc.eval(self.q, _lib.EPI_DEFECT, s=self.shift, Sb=self.S_base, Se=self.S_extra)


def smooth_ej(level: LevelState, n: int, omega: float = 1.0):
    """n sweeps of q <- q + omega B^-1 defect(q) (pmg.py:162-164)."""
    for _ in range(n):
        level.q = level.blocks.update(level.defect(), omega, level.q)


def smooth_rk(level: LevelState, n: int, cfl: float, alphas):
    """n sweeps of the pseudo-transient RK smoother: per sweep, from q0,
    stage j sets q <- q0 + alpha_j dtau_e defect(q) with the local step
    dtau_e = cfl / (s + lambda_e); each stage is one fused residual launch
    chain (oracle: solver_oracle.Pmg._smooth, "rk")."""
    d = level.disc
    dtau_e = d.rk_dtau(level.lam, level.shift, cfl)
    for _ in range(n):
        q0 = level.q
        for a in alphas:
            level.q = d.eval(level.q, _lib.EPI_RK, s=level.shift, Sb=level.S_base, Se=level.S_extra,
                             Q0=q0, dtau_e=dtau_e, alpha=a)


def smooth_mbnk(level: LevelState, rtol: float = 0.1, maxiter: int = 5):
    """One Newton update with the assembled block matrix and ILU0
    (pmg.py:167-175): GMRES(maxiter), one cycle, right-preconditioned by
    the block ILU0 of the level's block-sparse Jacobian."""
    r = level.defect()
    cfg = nk.KrylovConfig(kdim=maxiter, max_restarts=1, rtol=rtol)
    dq, _, _ = nk.gmres_solve(level.sparse.matvec, r, cfg, precond=lambda v: nk.ilu0_apply(level.ilu, v))
    level.q = lincomb((1.0, 1.0), (level.q, dq))


class PmgContext:
    """Level hierarchy, transfers and smoother state for one discretization."""

    def __init__(self, disc: Discretization, cfg: PmgPrecondConfig):
        self.disc = disc
        self.cfg = cfg
        h = cfg.hierarchy
        if disc.p != h.levels[0]:
            raise NotImplementedError("device pMG needs the discretization at the hierarchy top degree")
        self.levels = []
        for k, p in enumerate(h.levels):
            d = disc if k == 0 else disc.coarsen(p)
            self.levels.append(LevelState(d, nsweeps=h.smooth[k], smoother=h.smoothers[k]))
        self.tables = [_Transfer(self.levels[k].disc, self.levels[k + 1].disc)
                       for k in range(len(self.levels) - 1)]
        self.cycles_done = 0
        self.fallbacks = 0
        self.q_outer = None
        self.R_outer = None
        self.S_outer = None
        self.shift = 0.0
        # graph replay of precondition(): captured on the second call after a
        # prepare() (the first runs eagerly: lazy one-time setup in the library
        # must not happen under capture), dropped by the next prepare()
        self._graph = None
        self._graph_in = self._graph_out = None
        self._warm = False
        self.graph_replays = 0

    def prepare(self, q, shift: float):
        """Freeze the linearisation state and assemble the EJ blocks."""
        self._graph = None   # the cycle's arguments (state, shift, factors) change
        self._graph_in = self._graph_out = None
        q = to_device(q, self.disc.device)
        self.q_outer = q.clone()
        self.R_outer = self.levels[0].disc.eval(self.q_outer, _lib.EPI_R)
        self.S_outer = lincomb((shift, -1.0), (self.q_outer, self.R_outer))
        self.shift = shift
        qk = self.q_outer
        for k, lev in enumerate(self.levels):
            if k > 0:
                qk = self.tables[k - 1].restrict(qk)
            lev.shift = shift
            lev.frozen_q = qk
            lev.blocks = lev.sparse = lev.ilu = None   # free the old factors before assembling new ones
            if lev.smoother == "rk":   # matrix-free level: no element blocks
                lev.blocks = None
                lev.lam = lev.disc.rk_lambda(qk)
            else:
                lev.blocks = nk.assemble_element_blocks(lev.disc, qk, shift + self.cfg.smoother_shift,
                                                        keep_blocks=False, precision=self.cfg.block_precision)
            lev.sparse = lev.ilu = None
        raise_status()
        self.cycles_done = 0

    # -- smoother state (pmg.py:213-253) ----------------------------------

    def _effective_smoother(self, k: int) -> str:
        h = self.cfg.hierarchy
        if h.switch_after is not None and self.cycles_done >= h.switch_after:
            return "mbnk"
        return h.smoothers[k]

    def _ensure_sparse(self, lev: LevelState):
        """Block-sparse Jacobian at the frozen state and the level's current
        shift (no smoother_shift: that only damps the EJ blocks), and its
        block ILU0 -- built on first MBNK use after prepare()."""
        if lev.sparse is None:
            if active_partition() is not None:
                # block ILU0 is a global sequential sweep (newton_krylov.py:319-368)
                raise NotImplementedError("the MBNK smoother is not element-partitioned; use ej / rk")
            lev.sparse = nk.assemble_sparse_blocks(lev.disc, lev.frozen_q, lev.shift)
            lev.ilu = nk.ilu0_factor(lev.sparse)

    def _smooth(self, k: int):
        lev = self.levels[k]
        kind = self._effective_smoother(k)
        if kind == "rk":
            smooth_rk(lev, lev.nsweeps, self.cfg.rk_cfl, self.cfg.rk_alphas)
        elif kind == "ej":
            smooth_ej(lev, lev.nsweeps, self.cfg.omega)
        else:
            self._ensure_sparse(lev)
            for _ in range(lev.nsweeps):
                smooth_mbnk(lev, self.cfg.mbnk_rtol, self.cfg.mbnk_maxiter)

    def vcycle(self, k: int = 0):
        lev = self.levels[k]
        self._smooth(k)
        if k == len(self.levels) - 1:
            return
        d = lev.defect()
        coarse = self.levels[k + 1]
        T = self.tables[k]
        qb = T.restrict(lev.q)
        gd = T.restrict(d)
        coarse.q = qb.clone()
        coarse.S_base = coarse.F(qb)
        coarse.S_extra = gd
        self.vcycle(k + 1)
        lev.q = T.prolong_add(coarse.q, qb, lev.q.clone())
        self._smooth(k)

    # measured (tools/time_graph.py, profiles/r2/time_graph_r2v.jsonl): config 1 (16 K unknowns) 74.9 ->
    # 65.6 ms per step; even at 0.1-0.4 M; slower from 1.6 M (a capture per prepare(), the output copy)
    GRAPH_AUTO_DOFS = 65_536

    def _graphable(self) -> bool:
        """The V-cycles of precondition() are a fixed launch sequence between
        two prepare() calls when every level smooths with EJ or RK (MBNK runs
        a host-driven inner GMRES) on an unpartitioned mesh (the halo refresh
        is a host-issued collective)."""
        if self.cfg.graph == "off" or active_partition() is not None:
            return False
        h = self.cfg.hierarchy
        if h.switch_after is not None or any(s not in ("ej", "rk") for s in h.smoothers):
            return False
        return self.cfg.graph == "on" or self.disc.n_dofs <= self.GRAPH_AUTO_DOFS

    def _cycles(self, X) -> torch.Tensor:
        """m_max V-cycles on (s I - dR/dq) e = X from e = 0; returns e."""
        fine = self.levels[0]
        fine.q = self.q_outer.clone()
        fine.S_base = self.S_outer
        fine.S_extra = X
        for _ in range(self.cfg.m_max):
            self.vcycle()
        return lincomb((1.0, -1.0), (fine.q, self.q_outer))

    def precondition(self, X):
        """Approximate (s I - dR/dq)^-1 X by pseudo-time V-cycles (pmg.py:280-298).
        On small meshes the cycle is launch-bound (≈ 30 kernels of a few µs),
        so between two prepare() calls it is captured once into a CUDA graph
        and replayed: the same kernels in the same order, bit for bit."""
        is_np = not isinstance(X, torch.Tensor)
        X = to_device(X, self.disc.device)
        fine = self.levels[0]
        replay = self._graphable() and self._warm
        if replay:
            if self._graph is None:
                self._graph_in = torch.empty_like(X)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):   # a private pool per capture; prepare() drops it with the graph
                    self._graph_out = self._cycles(self._graph_in)
                self._graph = g
            self._graph_in.copy_(X)
            self._graph.replay()
            self.graph_replays += 1
            Y = self._graph_out
        else:
            Y = self._cycles(X)
            self._warm = True
        try:
            raise_status()
        except NonPhysicalStateError:
            self.fallbacks += 1
            if fine.blocks is None:   # RK fine level: the shift (diagonal) part of the EJ fallback
                Y = lincomb((1.0 / (self.shift + self.cfg.smoother_shift),), (X,))
            else:
                Y = fine.blocks.apply(X)
        else:
            if replay:
                Y = Y.clone()   # the graph's output buffer is rewritten by the next replay
        return Y.cpu().numpy() if is_np else Y


def pmg_precondition(X, ctx: PmgContext):
    return ctx.precondition(X)


def pmg_solve(ctx: PmgContext, q0, cfg: nk.PtcConfig, shift0: float = 0.0, const=0.0):
    """shift0 q - R(q) - const = 0 by PTC with one V-cycle per outer
    iteration (pmg.py:308-374)."""
    fine = ctx.levels[0]
    disc = fine.disc
    if isinstance(const, (np.ndarray, torch.Tensor)):
        cst = to_device(const, disc.device)
    elif float(const) != 0.0:
        cst = torch.full((disc.n_dofs,), float(const), dtype=torch.float64, device=disc.device)
    else:
        cst = 0.0

    def outer_F(q):
        return disc.eval(q, _lib.EPI_OUTER_F, s=shift0, Se=cst)

    q = to_device(q0, disc.device).clone()
    Fk = outer_F(q)
    n0 = nrm2(Fk)
    raise_status()
    stats = {"iters": 0, "gmres_iters": 0, "vcycles": 0, "converged": True, "aborted": False,
             "history": [(n0, 1.0, cfg.dtau_init)], "final_norm": n0}
    if n0 == 0.0 or (cfg.atol is not None and n0 <= cfg.atol):
        return q, stats
    dtau = cfg.dtau_init
    ctx.prepare(q, 1.0 / dtau + shift0)
    halved = False
    k = 0
    while k < cfg.max_iters:
        s_tot = 1.0 / dtau + shift0
        for lev in ctx.levels:
            lev.shift = s_tot
        fine.q = q.clone()
        fine.S_base = 0.0
        if isinstance(cst, torch.Tensor):
            fine.S_extra = lincomb((1.0 / dtau, 1.0), (q, cst))
        else:
            fine.S_extra = lincomb((1.0 / dtau,), (q,))
        try:
            ctx.vcycle()
            qn = fine.q
            Fn = outer_F(qn)
            nk_norm = nrm2(Fn)
            raise_status()
        except NonPhysicalStateError:
            if halved:
                stats["converged"] = False
                stats["aborted"] = True
                return q, stats
            halved = True
            dtau = 0.5 * dtau
            continue
        k += 1
        ctx.cycles_done += 1
        stats["iters"] = k
        stats["vcycles"] = k
        q, Fk = qn, Fn
        if cfg.ser:
            prev = stats["history"][-1][0]
            dtau = nk.ser_update(dtau, prev, nk_norm, cfg.dtau_max, cfg.ser_as_printed)
        stats["history"].append((nk_norm, nk_norm / n0 if n0 else 0.0, dtau))
        stats["final_norm"] = nk_norm
        if nk_norm / n0 <= cfg.rtol or (cfg.atol is not None and nk_norm <= cfg.atol):
            return q, stats
        if cfg.refresh_every and k % cfg.refresh_every == 0:
            ctx.prepare(q, 1.0 / dtau + shift0)
    stats["converged"] = False
    return q, stats
