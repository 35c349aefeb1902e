"""Implicit driver glue on the device path -- drop-in for
pmgflow.harness.ImplicitDriver (``harness.py:277-369``).

``ImplicitDriver(disc, cfg)`` accepts the reference's flat config keys
(``ptc.*``, ``gmres.*``, ``pmg.*``, ``case.precond``) as a dict or an
object with ``__getitem__``; missing keys take the reference defaults
(harness.py:45-113).  Stage records mirror StageRecord / SolverStats
(harness.py:175-207).  ``run_case`` (harness.py:385-487) runs a configured
case on the device and writes the reference's CSV artifacts (residual,
stats, forces, summary); config text parsing follows
``parse_config_text`` (:139-165).  Mesh files, p-adaptation, the OOA /
preconditioner studies and the CLI are outside the hot-path scope.
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass, field
from pathlib import Path

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
    "gmres.kdim": 30, "gmres.max_restarts": 10, "gmres.rtol": 1e-4, "gmres.ortho": "mgs",
    "pmg.levels": "3-1", "pmg.smooth": "2", "pmg.smoother": "ej", "pmg.switch_after": None,
    "pmg.mbnk.rtol": 0.1, "pmg.mbnk.maxiter": 5, "pmg.smoother_shift": 0.0,
    "pmg.rk.cfl": 1.5, "pmg.rk.stages": "0.25,0.3333333333333333,0.5,1.0", "pmg.block_precision": "fp64",
    "pmg.graph": "auto", "case.precond": "ej",
}


def pmg_precond_config(cfg) -> "pmg_mod.PmgPrecondConfig":
    """pmg.* keys -> PmgPrecondConfig.  pmg.rk.* configure the pseudo-transient
    RK smoother (smoother kind "rk", an extension: the reference knows only
    ej / mbnk, harness.py:97)."""
    h = pmg_mod.PHierarchy.parse(cfg["pmg.levels"], cfg["pmg.smooth"], cfg["pmg.smoother"],
                                 cfg["pmg.switch_after"])
    alphas = tuple(float(a) for a in str(cfg["pmg.rk.stages"]).split(","))
    return pmg_mod.PmgPrecondConfig(h, mbnk_rtol=cfg["pmg.mbnk.rtol"], mbnk_maxiter=cfg["pmg.mbnk.maxiter"],
                                    smoother_shift=cfg["pmg.smoother_shift"],
                                    rk_cfl=float(cfg["pmg.rk.cfl"]),
                                    rk_alphas=alphas,
                                    block_precision=str(cfg["pmg.block_precision"]),
                                    graph=str(cfg["pmg.graph"]))


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
                           rtol=cfg["gmres.rtol"], ortho=cfg["gmres.ortho"])


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
            self.ctx = pmg_mod.PmgContext(disc, pmg_precond_config(cfg))
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


# ---------------------------------------------------------------------------
# configured cases and their artifacts (harness.py:28-168, 213-247, 375-487)

class ConfigError(Exception):
    pass


def _as_bool(s: str) -> bool:
    t = str(s).strip().lower()
    if t in ("true", "yes", "on", "1"):
        return True
    if t in ("false", "no", "off", "0"):
        return False
    raise ValueError(f"not a boolean: {s!r}")


SCHEMA = {
    "mesh.kind": (str, "box"), "mesh.path": (str, None), "mesh.nx": (int, 4), "mesh.ny": (int, 4),
    "mesh.lx": (float, 1.0), "mesh.ly": (float, 1.0), "mesh.periodic": (_as_bool, False),
    "mesh.tag": (str, "far-field"), "mesh.n_circ": (int, 40), "mesh.n_rad": (int, 20),
    "mesh.r_wall": (float, 0.5), "mesh.r_far": (float, 60.0), "mesh.stretch": (float, 1.25),
    "mesh.wall_tag": (str, "wall-adiabatic"),
    "equation.kind": (str, "euler"), "equation.mach": (float, 0.1), "equation.reynolds": (float, 100.0),
    "equation.ref_length": (float, 1.0), "equation.gamma": (float, 1.4), "equation.prandtl": (float, 0.72),
    "equation.advection_x": (float, 1.0), "equation.advection_y": (float, 0.0),
    "equation.diffusivity": (float, 0.0),
    "case.degree": (int, 2), "case.scheme": (str, "esdirk2"), "case.dt": (float, 0.1), "case.steps": (int, 1),
    "case.steady": (_as_bool, False), "case.solver": (str, "jfnk"), "case.precond": (str, "ej"),
    "case.init": (str, "free-stream"), "case.seed": (int, 0),
    "ptc.dtau_init": (float, 1e-3), "ptc.dtau_max": (float, 1e12), "ptc.max_iters": (int, 100),
    "ptc.rtol": (float, 1e-4), "ptc.atol": (float, None), "ptc.ser": (_as_bool, True),
    "ptc.ser_as_printed": (_as_bool, False), "ptc.refresh_every_n_ptc": (int, 0), "ptc.max_halvings": (int, 8),
    "gmres.kdim": (int, 30), "gmres.max_restarts": (int, 10), "gmres.rtol": (float, 1e-4),
    "gmres.ortho": (str, "mgs"),
    "pmg.levels": (str, "3-1"), "pmg.smooth": (str, "2"), "pmg.smoother": (str, "ej"),
    "pmg.switch_after": (int, None), "pmg.mbnk.rtol": (float, 0.1), "pmg.mbnk.maxiter": (int, 5),
    "pmg.smoother_shift": (float, 0.0), "pmg.rk.cfl": (float, 1.5),
    "pmg.rk.stages": (str, "0.25,0.3333333333333333,0.5,1.0"), "pmg.block_precision": (str, "fp64"), "pmg.graph": (str, "auto"),
    "adapt.enable": (_as_bool, False), "adapt.variable": (str, "momentum-x"), "adapt.nu_max": (float, 0.2),
    "adapt.nu_min": (float, 0.001), "adapt.p_min": (int, 1), "adapt.p_max": (int, 4),
    "adapt.every_n_steps": (int, 10),
    "ooa.mode": (str, "spatial"), "ooa.case": (str, "advected-sine"),
}
_VALID_CHOICES = {
    "mesh.kind": ("box", "cylinder", "file"),
    "equation.kind": ("euler", "navier-stokes", "advection-diffusion"),
    "case.scheme": ("esdirk2", "esdirk3", "esdirk4", "row2", "row4", "ros4l"),
    "gmres.ortho": ("mgs", "cgs2"),
    "case.solver": ("jfnk", "pmg-solver"),
    "case.precond": ("ej", "pmg", "none"),
    "pmg.block_precision": ("fp64", "fp32"),
    "pmg.graph": ("auto", "on", "off"),
    "case.init": ("free-stream", "zero"),
    "ooa.mode": ("spatial", "temporal"),
    "ooa.case": ("advected-sine", "vortex"),
}


@dataclass
class CaseConfig:
    values: dict

    def __getitem__(self, key):
        return self.values[key]

    def get(self, key, default=None):
        v = self.values.get(key)
        return default if v is None else v


def parse_config_text(text: str, overrides: dict | None = None) -> CaseConfig:
    """'section.key = value' lines, '#' comments, typed and validated
    against SCHEMA (harness.py:139-165)."""
    values = {k: default for k, (_, default) in SCHEMA.items()}
    entries = {}
    for ln, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {ln}: expected 'section.key = value'")
        key, val = (t.strip() for t in line.split("=", 1))
        entries[key] = (val, ln)
    for k, v in (overrides or {}).items():
        entries[k] = (str(v), 0)
    for key, (val, ln) in entries.items():
        if key not in SCHEMA:
            raise ConfigError(f"unknown config key {key!r} (line {ln})")
        try:
            values[key] = SCHEMA[key][0](val)
        except ValueError as exc:
            raise ConfigError(f"bad value for {key!r}: {exc}") from None
    for key, choices in _VALID_CHOICES.items():
        if values[key] is not None and values[key] not in choices:
            raise ConfigError(f"{key} must be one of {choices}, got {values[key]!r}")
    return CaseConfig(values)


def load_config(path) -> CaseConfig:
    return parse_config_text(Path(path).read_text())


def mesh_from_config(cfg):
    from .mesh import generate_box, generate_cylinder_omesh
    kind = cfg["mesh.kind"]
    if kind == "box":
        return generate_box(cfg["mesh.nx"], cfg["mesh.ny"], cfg["mesh.lx"], cfg["mesh.ly"],
                            periodic=cfg["mesh.periodic"], tag=cfg["mesh.tag"])
    if kind == "cylinder":
        return generate_cylinder_omesh(cfg["mesh.n_circ"], cfg["mesh.n_rad"], cfg["mesh.r_wall"],
                                       cfg["mesh.r_far"], cfg["mesh.stretch"], wall_tag=cfg["mesh.wall_tag"])
    raise ConfigError("mesh.kind = file: mesh files are not on the device path (pass a Mesh instead)")


def equation_from_config(cfg):
    from .equation import EquationSpec
    try:
        return EquationSpec(kind=cfg["equation.kind"], mach=cfg["equation.mach"],
                            reynolds=cfg["equation.reynolds"], ref_length=cfg["equation.ref_length"],
                            gamma=cfg["equation.gamma"], prandtl=cfg["equation.prandtl"],
                            advection=(cfg["equation.advection_x"], cfg["equation.advection_y"]),
                            diffusivity=cfg["equation.diffusivity"])
    except ValueError as exc:
        raise ConfigError(str(exc)) from None


def initial_field(disc: Discretization, cfg):
    if cfg["case.init"] == "zero" or disc.eqn.kind == "advection-diffusion":
        return disc.new_field().data
    return disc.free_stream_field().data


def _write_csv(path: Path, header_comment: str, columns, rows):
    with open(path, "w", newline="") as f:
        f.write(f"# {header_comment}\n")
        w = csv.writer(f)
        w.writerow(columns)
        for row in rows:
            w.writerow([repr(float(v)) if isinstance(v, float) else v for v in row])


def run_case(cfg, out_dir, mesh=None) -> dict:
    """Run one configured case on the device; returns a summary dict and
    writes residual.csv, stats.csv, forces.csv (wall cases) and summary.csv
    (harness.py:385-487).  ``mesh`` overrides ``mesh.*``."""
    if cfg["adapt.enable"]:
        raise NotImplementedError("p-adaptation (mixed degrees) is not on the device path (SURVEY 8(f))")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    mesh = mesh if mesh is not None else mesh_from_config(cfg)
    eqn = equation_from_config(cfg)
    disc = Discretization(mesh, cfg["case.degree"], eqn)
    scheme = ti.get_scheme(cfg["case.scheme"])
    driver = ImplicitDriver(disc, cfg)
    q = initial_field(disc, cfg)
    dt = cfg["case.dt"]
    has_walls = any(str(t).startswith("wall") for t in mesh.boundary_tags) and eqn.kind != "advection-diffusion"
    forces = []
    t_begin = time.perf_counter()
    converged = True
    try:
        if cfg["case.steady"]:
            if cfg["case.solver"] == "pmg-solver":
                ctx = pmg_mod.PmgContext(disc, pmg_precond_config(cfg))
                q, stats = pmg_mod.pmg_solve(ctx, q, driver.ptc)
                driver.stats.records.append(StageRecord(0, 0, stats["iters"], 0, stats["vcycles"], 0.0))
                for it, (absr, relr, dtau) in enumerate(stats["history"]):
                    driver.stats.residual_log.append((0, 0, it, absr, relr, dtau))
            else:
                q, stats = driver.solve_stage(ti.StageProblem(disc.residual, steady=True), q)
            converged = stats["converged"]
            final_norm = stats["final_norm"]
        else:
            for step in range(cfg["case.steps"]):
                driver._step = step
                q, _ = driver.step(q, dt, scheme)
                if has_walls:
                    fd, fl, cd, cl = disc.compute_forces(q)
                    forces.append(((step + 1) * dt, cd, cl))
            final_norm = float(nrm2(disc.residual(to_device(q, disc.device))))
    except RuntimeError as exc:
        converged = False
        final_norm = float("nan")
        summary_error = str(exc)
    else:
        summary_error = ""
    runtime = time.perf_counter() - t_begin
    driver.stats.total_runtime = runtime
    st = driver.stats
    _write_csv(out / "residual.csv", "pmgflow residual v1",
               ("step", "stage", "iter", "absolute", "relative", "dtau"), st.residual_log)
    _write_csv(out / "stats.csv", "pmgflow stats v1",
               ("step", "stage", "n_ptc", "n_gmres", "n_vcycles", "wall_time"),
               [(r.step, r.stage, r.ptc_iters, r.gmres_iters, r.vcycles, r.wall_time) for r in st.records])
    if has_walls and forces:
        _write_csv(out / "forces.csv", "pmgflow forces v1", ("t", "cd", "cl"), forces)
    summary = {"converged": converged, "final_residual": final_norm, "n_ptc_avg": st.n_ptc_avg,
               "n_gmres_avg": st.n_gmres_avg, "kdim": st.kdim, "runtime": runtime, "error": summary_error,
               "stats": st, "q": q.cpu().numpy() if hasattr(q, "cpu") else q, "disc": disc}
    _write_csv(out / "summary.csv", "pmgflow summary v1",
               ("converged", "final_residual", "n_ptc_avg", "n_gmres_avg", "kdim", "runtime"),
               [(int(converged), final_norm, st.n_ptc_avg, st.n_gmres_avg, st.kdim, runtime)])
    return summary
