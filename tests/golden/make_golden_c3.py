"""Golden pmg_solve history at the full BASELINE config-3 size, produced
by the REFERENCE.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_c3.py

BASELINE config 3 (128 x 128 periodic box, p = 4, NS at Ma 1e-3, Re 500,
density bump + 1e-6 velocity noise): the reference's nonlinear pMG solver
(pmg.py:308-374) over the full hierarchy p{4-3-2-1-0} with element-Jacobi
smoothing on every level (smoother_shift 1e3, the bench's setting), PTC
dtau_init 0.1, for the first three outer iterations.  The reference cannot
reach BASELINE's 10-order drop; the residual history of these
iterations and the state after them (every 16th element in full, and
per-variable sums over all elements) are what the device must reproduce
(tests/test_gpu_fullsize_oracle.py).  Output: golden_c3.npz.
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

from pmgflow import mesh as rmesh  # noqa: E402
from pmgflow import newton_krylov as rnk  # noqa: E402
from pmgflow import pmg as rpmg  # noqa: E402
from pmgflow import spatial as rsp  # noqa: E402

from make_golden import ref_eqn  # noqa: E402
from paper_2202_09733_b200 import cases  # noqa: E402

ITERS = 3


def main():
    c = cases.config(3)
    d = rsp.Discretization(rmesh.generate_box(128, 128, 10.0, 10.0, periodic=True), 4, ref_eqn(c.eqn))
    h = rpmg.PHierarchy.parse(c.levels, "2", "ej")
    ctx = rpmg.PmgContext(d, rpmg.PmgPrecondConfig(h, smoother_shift=c.extra["smoother_shift"]))
    cfg = rnk.PtcConfig(dtau_init=0.1, dtau_max=1e12, max_iters=ITERS, rtol=1e-14)
    t0 = time.perf_counter()
    q, st = rpmg.pmg_solve(ctx, c.q0, cfg)
    wall = time.perf_counter() - t0
    hist = np.array(st["history"])
    print("history", hist.tolist(), f"{wall:.1f}s", flush=True)
    # the state: every 16th element in full, plus per-variable sums of all
    Q = q.reshape(c.mesh.n_elements, -1)
    np.savez_compressed(HERE / "golden_c3.npz", history=hist, iters=np.array(st["iters"]), wall_s=np.array(wall),
                        q_sub=Q[::16].copy(), sub_stride=np.array(16),
                        q_sum=Q.reshape(len(Q), -1, 4).sum(axis=(0, 1)),
                        q_abs_sum=np.abs(Q.reshape(len(Q), -1, 4)).sum(axis=(0, 1)))


if __name__ == "__main__":
    main()
