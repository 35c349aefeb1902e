"""Golden run_case artifacts (harness.py:385-487), made by running the
REFERENCE pmgflow in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_harness.py

Small cylinder cases with walls (ESDIRK2 / ROW2, EJ and pMG
preconditioners); the CSV files are stored as text in
tests/golden/golden_harness.npz."""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from pmgflow import harness as rh  # noqa: E402

CASES = {
    "cyl_euler_esdirk2_ej": """
mesh.kind = cylinder
mesh.n_circ = 12
mesh.n_rad = 4
mesh.r_far = 8.0
mesh.stretch = 1.3
equation.kind = euler
equation.mach = 0.3
case.degree = 1
case.scheme = esdirk2
case.dt = 0.05
case.steps = 2
case.precond = ej
ptc.dtau_init = 0.05
gmres.rtol = 1e-3
""",
    "cyl_ns_row2_ej": """
mesh.kind = cylinder
mesh.n_circ = 12
mesh.n_rad = 4
mesh.r_far = 8.0
mesh.stretch = 1.3
equation.kind = navier-stokes
equation.mach = 0.3
equation.reynolds = 200
case.degree = 1
case.scheme = row2
case.dt = 0.02
case.steps = 2
case.precond = ej
gmres.rtol = 1e-4
""",
    "cyl_ns_esdirk2_pmg": """
mesh.kind = cylinder
mesh.n_circ = 12
mesh.n_rad = 4
mesh.r_far = 8.0
mesh.stretch = 1.3
equation.kind = navier-stokes
equation.mach = 0.3
equation.reynolds = 200
case.degree = 2
case.scheme = esdirk2
case.dt = 0.05
case.steps = 1
case.precond = pmg
pmg.levels = 2-1
pmg.smoother_shift = 20
ptc.dtau_init = 0.05
gmres.rtol = 1e-3
""",
}


def main():
    out = {}
    for name, text in CASES.items():
        with tempfile.TemporaryDirectory() as tmp:
            summ = rh.run_case(rh.parse_config_text(text), tmp)
            for fn in ("residual", "stats", "forces", "summary"):
                f = Path(tmp) / f"{fn}.csv"
                out[f"{name}/{fn}"] = np.array(f.read_text() if f.exists() else "")
        out[f"{name}/cfg"] = np.array(text)
        out[f"{name}/q"] = summ["q"]
        print(name, "converged", summ["converged"], "ptc", summ["n_ptc_avg"], "gmres", summ["n_gmres_avg"])
    np.savez_compressed(HERE / "golden_harness.npz", **out)


if __name__ == "__main__":
    main()
