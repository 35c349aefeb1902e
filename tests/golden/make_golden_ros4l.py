"""Golden vectors for the derived 4-stage ROW tableau (ros4l), produced by
the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_ros4l.py

BASELINE config 4 names "a 4-stage ROW method"; the reference's row4 is the
six-stage RODASP (time_integration.py:80-102).  Its ``row_step``
(:171-197) takes any StageScheme, so the tableau derived in
paper_2202_09733_b200.time_integration._ros4l is injected into the
reference's own stepper and ImplicitDriver.solve_linear (harness.py:337)
here, on the config-1 case; the reference's ``validate_tableau`` /
``stability_function`` (:200-251) results are recorded alongside.
Output: tests/golden/golden_ros4l.npz.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from pmgflow import harness as hz  # noqa: E402
from pmgflow import mesh as rmesh  # noqa: E402
from pmgflow import spatial as rsp  # noqa: E402
from pmgflow import time_integration as rti  # noqa: E402

from make_golden import GmresLog, ref_eqn  # noqa: E402
from paper_2202_09733_b200 import cases  # noqa: E402
from paper_2202_09733_b200 import time_integration as ti  # noqa: E402


def ref_scheme():
    s = ti.get_scheme("ros4l")
    return rti.StageScheme(s.name, s.kind, s.order, s.a.copy(), s.b.copy(), s.c.copy(), s.cmat.copy(), s.gamma)


def main():
    out = {}
    sch = ref_scheme()
    rep = rti.validate_tableau(sch)
    out["tableau/a"] = sch.a
    out["tableau/cmat"] = sch.cmat
    out["tableau/m"] = sch.b
    out["tableau/checks"] = np.array([bool(v) for v in rep.values()])
    out["tableau/check_names"] = np.array(list(rep.keys()))
    zs = np.array([-1e6, -10.0, -1.0, 1j, 10j, 100j, -1 + 1j])
    out["tableau/z"] = zs
    out["tableau/R"] = np.array([rti.stability_function(sch, z) for z in zs])
    print(rep)

    c = cases.config(1)
    d = rsp.Discretization(rmesh.generate_box(16, 16, 10.0, 10.0, periodic=True), 3, ref_eqn(c.eqn))
    cfg = hz.parse_config_text("""
case.precond = pmg
pmg.levels = 3-2
pmg.smooth = 2
pmg.smoother_shift = 50
gmres.kdim = 30
gmres.rtol = 1e-3
""")
    drv = hz.ImplicitDriver(d, cfg)
    t0 = time.perf_counter()
    with GmresLog() as log:
        Rl = d.residual(c.q0)
        qn, info = rti.row_step(c.q0, c.dt, sch, d.residual, drv.solve_linear(c.q0, Rl))
    wall = time.perf_counter() - t0
    out["c1/ros4l/q1"] = qn
    out["c1/ros4l/gmres_counts"] = np.array(log.counts)
    out["c1/ros4l/wall_s"] = np.array(wall)
    print("ros4l gmres per solve", log.counts, f"{wall:.2f}s")
    np.savez_compressed(HERE / "golden_ros4l.npz", **out)


if __name__ == "__main__":
    main()
