"""Equation specification and the non-physical-state exception.

Same fields, defaults, validation and derived quantities as the
reference's ``EquationSpec`` (spatial.py:35-88) and
``NonPhysicalStateError`` (spatial.py:27-32), so that host code written
against the reference constructs the device discretization unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KIND_CODE = {"euler": 0, "navier-stokes": 1, "advection-diffusion": 2}


class NonPhysicalStateError(Exception):
    """Negative density or pressure met during a flux evaluation."""

    def __init__(self, element: int, what: str = "state"):
        self.element = int(element)
        self.what = what
        super().__init__(f"non-physical {what} in element {self.element}")


@dataclass(frozen=True)
class EquationSpec:
    kind: str = "euler"
    mach: float = 0.1
    reynolds: float = 100.0
    ref_length: float = 1.0
    gamma: float = 1.4
    prandtl: float = 0.72
    advection: tuple = (1.0, 0.0)
    diffusivity: float = 0.0
    # interface schemes: the reference has Roe + BR1 only (spatial.py:113-163,
    # 536-603); "rusanov" / "ldg" are the BASELINE configs' choices (SURVEY
    # 8.0), parity-pinned to the oracle only
    riemann: str = "roe"
    viscous_scheme: str = "br1"
    # temperature T = p / rho held by "wall-isothermal" faces (BASELINE
    # config 4's no-slip isothermal wall; not in the reference, whose walls
    # are adiabatic / slip, spatial.py:183-203).  None = free-stream T.
    wall_temperature: float | None = None

    def __post_init__(self):
        if self.kind not in KIND_CODE:
            raise ValueError(f"unknown equation kind {self.kind!r}")
        if self.riemann not in ("roe", "rusanov"):
            raise ValueError(f"unknown Riemann flux {self.riemann!r}")
        if self.viscous_scheme not in ("br1", "ldg"):
            raise ValueError(f"unknown viscous scheme {self.viscous_scheme!r}")
        if self.wall_temperature is not None and not self.wall_temperature > 0:
            raise ValueError("wall temperature must be positive")
        if self.kind != "advection-diffusion" and self.mach <= 0:
            raise ValueError("Mach number must be positive")
        if self.kind == "navier-stokes" and self.reynolds <= 0:
            raise ValueError("Reynolds number must be positive")

    @property
    def nvars(self) -> int:
        return 1 if self.kind == "advection-diffusion" else 4

    @property
    def viscous(self) -> bool:
        if self.kind == "navier-stokes":
            return True
        return self.kind == "advection-diffusion" and self.diffusivity > 0.0

    @property
    def mu(self) -> float:
        return self.ref_length / self.reynolds if self.kind == "navier-stokes" else 0.0

    @property
    def heat_conductivity(self) -> float:
        g = self.gamma
        return self.mu * g / ((g - 1.0) * self.prandtl)

    @property
    def t_wall(self) -> float:
        """Isothermal wall temperature (p / rho); free-stream 1/(gamma Ma^2)."""
        if self.wall_temperature is not None:
            return float(self.wall_temperature)
        return 0.0 if self.kind == "advection-diffusion" else 1.0 / (self.gamma * self.mach ** 2)

    def free_stream(self) -> np.ndarray:
        if self.kind == "advection-diffusion":
            return np.zeros(1)
        p = 1.0 / (self.gamma * self.mach ** 2)
        return np.array([1.0, 1.0, 0.0, p / (self.gamma - 1.0) + 0.5])
