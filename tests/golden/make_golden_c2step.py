"""Golden ESDIRK3 step at the bench's config-2 settings, produced by the REFERENCE.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_c2step.py

BASELINE config 2 (NS, Ma 0.5, Re 1000, vortex + 1e-6 noise, p{4-2},
GMRES(30), rtol 1e-3) on a 48 x 48 version of its mesh with the bench's
settings: ESDIRK3 (the derived tableau injected into the reference's own
``esdirk_step``, time_integration.py:144-168), pmg.smoother_shift 5000,
ptc.dtau_init = dt, dt = 50 dt_conv.  The reference's ImplicitDriver
(harness.py:277-369) runs the step; the GMRES count of every linear
solve, the PTC counts and the new state are recorded in
golden_c2step.npz for tests/test_gpu_fullsize_oracle.py.
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
from make_golden_esdirk3 import ref_scheme  # noqa: E402
from paper_2202_09733_b200 import cases  # noqa: E402

NX = 48


def main():
    c = cases.config(2, nx=NX)
    d = rsp.Discretization(rmesh.generate_box(NX, NX, 10.0, 10.0, periodic=True), 4, ref_eqn(c.eqn))
    cfg = hz.parse_config_text(f"""
case.precond = pmg
pmg.levels = 4-2
pmg.smooth = 2
pmg.smoother_shift = 5000
gmres.kdim = 30
gmres.rtol = 1e-3
ptc.dtau_init = {c.dt!r}
ptc.rtol = 1e-4
""")
    drv = hz.ImplicitDriver(d, cfg)
    t0 = time.perf_counter()
    with GmresLog() as log:
        qn, info = rti.esdirk_step(c.q0, c.dt, ref_scheme(), d.residual, drv.solve_stage)
    wall = time.perf_counter() - t0
    import hashlib
    out = {"q0_sha256": np.array(hashlib.sha256(c.q0.tobytes()).hexdigest()), "dt": np.array(c.dt), "q1": qn, "gmres_counts": np.array(log.counts),
           "ptc_iters": np.array([i["iters"] for i in info]), "wall_s": np.array(wall)}
    print("gmres per solve", log.counts, "ptc", [i["iters"] for i in info], f"{wall:.1f}s", flush=True)
    np.savez_compressed(HERE / "golden_c2step.npz", **out)


if __name__ == "__main__":
    main()
