"""Implicit driver glue on the device path -- drop-in for
pmgflow.harness.ImplicitDriver (``harness.py:277-369``).

``ImplicitDriver(disc, cfg)`` accepts the reference's flat config keys
(``ptc.*``, ``gmres.*``, ``pmg.*``, ``case.precond``) as a dict or an
object with ``__getitem__``; missing keys take the reference defaults
(harness.py:45-113).  Stage records mirror StageRecord / SolverStats
(harness.py:175-207).  Config files, CSV artifacts, studies and the CLI
(the rest of harness.py) are outside the hot-path scope.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import newton_krylov as nk
from . import pmg as pmg_mod
from . import time_integration as ti
from .spatial import Discretization
from .vec import nrm2, to_device

DEFAULTS = {
    "ptc.dtau_init": 1e-3, "ptc.dtau_max": 1e12, "ptc.max_iters": 100, "ptc.rtol": 1e-4,
    "ptc.atol": None, "ptc.ser": True, "ptc.ser_as_printed": False, "ptc.refresh_every_n_ptc": 0,
    "ptc.max_halvings": 8,
    "gmres.kdim": 30, "gmres.max_restarts": 10, "gmres.rtol": 1e-4,
    "pmg.levels": "3-1", "pmg.smooth": "2", "pmg.smoother": "ej", "pmg.switch_after": None,
    "pmg.mbnk.rtol": 0.1, "pmg.mbnk.maxiter": 5, "pmg.smoother_shift": 0.0,
    "case.precond": "ej",
}


@dataclass
class StageRecord:
    step: int
    stage: int
    ptc_iters: int
    gmres_iters: int
    vcycles: int
    wall_time: float


@dataclass
class SolverStats:
    kdim: int
    records: list = field(default_factory=list)
    total_runtime: float = 0.0
    residual_log: list = field(default_factory=list)
    fallbacks: int = 0

    @property
    def n_stages(self):
        return len(self.records)

    @property
    def n_ptc_avg(self):
        return sum(r.ptc_iters for r in self.records) / len(self.records) if self.records else 0.0

    @property
    def n_gmres_avg(self):
        return sum(r.gmres_iters for r in self.records) / len(self.records) if self.records else 0.0


class _Cfg:
    def __init__(self, values):
        self.values = dict(DEFAULTS)
        if values is not None:
            src = values.values if hasattr(values, "values") and isinstance(values.values, dict) else values
            self.values.update({k: v for k, v in dict(src).items() if v is not None or k in DEFAULTS})

    def __getitem__(self, k):
        return self.values[k]


def ptc_config(cfg) -> nk.PtcConfig:
    return nk.PtcConfig(dtau_init=cfg["ptc.dtau_init"], dtau_max=cfg["ptc.dtau_max"],
                        max_iters=cfg["ptc.max_iters"], rtol=cfg["ptc.rtol"], atol=cfg["ptc.atol"],
                        ser=cfg["ptc.ser"], ser_as_printed=cfg["ptc.ser_as_printed"],
                        refresh_every=cfg["ptc.refresh_every_n_ptc"], max_halvings=cfg["ptc.max_halvings"])


def krylov_config(cfg) -> nk.KrylovConfig:
    return nk.KrylovConfig(kdim=cfg["gmres.kdim"], max_restarts=cfg["gmres.max_restarts"],
                           rtol=cfg["gmres.rtol"])


class ImplicitDriver:
    """Stage solvers (ESDIRK: PTC + JFNK-GMRES; ROW: one GMRES per stage)
    with an EJ or pMG preconditioner, all on the device."""

    def __init__(self, disc: Discretization, cfg=None):
        cfg = _Cfg(cfg)
        self.disc = disc
        self.cfg = cfg
        self.ptc = ptc_config(cfg)
        self.krylov = krylov_config(cfg)
        self.precond = cfg["case.precond"]
        self.stats = SolverStats(kdim=self.krylov.kdim)
        self.ctx = None
        if self.precond == "pmg":
            h = pmg_mod.PHierarchy.parse(cfg["pmg.levels"], cfg["pmg.smooth"], cfg["pmg.smoother"],
                                         cfg["pmg.switch_after"])
            pc = pmg_mod.PmgPrecondConfig(h, mbnk_rtol=cfg["pmg.mbnk.rtol"], mbnk_maxiter=cfg["pmg.mbnk.maxiter"],
                                          smoother_shift=cfg["pmg.smoother_shift"])
            self.ctx = pmg_mod.PmgContext(disc, pc)
        self._step = 0
        self._stage = 0

    def _precond_factory(self, shift0: float):
        if self.precond == "none":
            return None
        if self.precond == "ej":
            def factory(q, dtau):
                bj = nk.assemble_element_blocks(self.disc, q, shift0 + 1.0 / dtau, keep_blocks=False)
                return bj.apply
            return factory

        def factory(q, dtau):
            self.ctx.prepare(q, shift0 + 1.0 / dtau)
            return self.ctx.precondition
        return factory

    def solve_stage(self, prob: ti.StageProblem, q0):
        t0 = time.perf_counter()
        F = ti.StageFunction(prob)
        cycles0 = self.ctx.cycles_done if self.ctx is not None else 0
        q, stats = nk.ptc_solve(F, q0, self.ptc, self.krylov,
                                precond_factory=self._precond_factory(prob.shift))
        wall = time.perf_counter() - t0
        cycles = (self.ctx.cycles_done - cycles0) if self.ctx is not None else 0
        self.stats.records.append(StageRecord(self._step, self._stage, stats["iters"],
                                              stats["gmres_iters"], cycles, wall))
        for it, (absr, relr, dtau) in enumerate(stats["history"]):
            self.stats.residual_log.append((self._step, self._stage, it, absr, relr, dtau))
        if self.ctx is not None:
            self.stats.fallbacks = self.ctx.fallbacks
        return q, stats

    def solve_linear(self, q_lin, R_lin):
        prepared = {}
        q_lin = to_device(q_lin, self.disc.device)
        R_lin = to_device(R_lin, self.disc.device)

        def solve(rhs, sigma, stage):
            t0 = time.perf_counter()
            if "P" not in prepared:
                if self.precond == "ej":
                    bj = nk.assemble_element_blocks(self.disc, q_lin, sigma, keep_blocks=False)
                    prepared["P"] = bj.apply
                elif self.precond == "pmg":
                    self.ctx.prepare(q_lin, sigma)
                    prepared["P"] = self.ctx.precondition
                else:
                    prepared["P"] = None

            def matvec(v):
                return nk.jfnk_matvec(v, q_lin, R_lin, self.disc.residual, sigma, check_zero=False, sync=False)

            Y, iters, relres = nk.gmres_solve(matvec, rhs, self.krylov, precond=prepared["P"])
            wall = time.perf_counter() - t0
            converged = relres <= self.krylov.rtol
            self.stats.records.append(StageRecord(self._step, stage, 0, iters, 0, wall))
            self.stats.residual_log.append((self._step, stage, iters, relres * nrm2(to_device(rhs)), relres, 0.0))
            return Y, {"converged": bool(converged), "iters": iters, "relres": relres}
        return solve

    # convenience: one physical step of the configured scheme
    def step(self, q, dt: float, scheme: ti.StageScheme):
        if scheme.kind == "esdirk":
            counter = [0]

            def solve_stage(prob, q0):
                counter[0] += 1
                self._stage = counter[0]
                return self.solve_stage(prob, q0)
            return ti.esdirk_step(q, dt, scheme, self.disc.residual, solve_stage)
        R_lin = self.disc.residual(to_device(q, self.disc.device))
        return ti.row_step(q, dt, scheme, self.disc.residual, self.solve_linear(q, R_lin))
