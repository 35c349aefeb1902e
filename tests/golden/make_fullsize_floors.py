"""Rounding floors of the *reference itself* at the BASELINE full sizes.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_floors.py

At 256^2 and beyond, two correct float64 evaluations of R that order their
operations differently disagree by far more than the north star's 1e-12:
the reference and the oracle differ by 1.2e-9 (max-norm, relative) at
config 2.  So the full-size parity tests measure every float64 evaluation
against one extended-precision "truth" -- the oracle's algorithm evaluated
in x87 long double (64-bit significand) on the same float64 operators,
geometry and inputs (``OracleDisc(..., dtype=np.longdouble)``) -- and
require the device to be at least as close to it as the reference's own
float64 arithmetic.  This script runs the reference's
``Discretization.residual`` (pkg/src/pmgflow/spatial.py:501-570) and its
FD Jacobian-vector product (newton_krylov.py:71-76) at configs 2-5 and
records their distance to that truth in ``fullsize_floors.json`` (a few
numbers; the reference cannot travel to the GPU box).
"""

from __future__ import annotations

import gc
import json
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
from pmgflow import spatial as rsp  # noqa: E402

from make_golden import ref_eqn  # noqa: E402
from oracle.fr_oracle import OracleDisc  # noqa: E402
from paper_2202_09733_b200 import cases  # noqa: E402

JV_SHIFT, JV_SEED = 3.0, 7


def reference_case(k):
    """(case, reference Discretization) for BASELINE config k.  Config 4's
    no-slip wall is isothermal here, which the reference lacks: its floor is
    measured on the same stretched channel with the reference's adiabatic
    wall (same geometry, same operators)."""
    import dataclasses

    from paper_2202_09733_b200 import mesh as mm
    c = cases.config(k)
    if k != 4:
        n = int(round(np.sqrt(c.mesh.n_elements)))
        return c, rsp.Discretization(rmesh.generate_box(n, n, 10.0, 10.0, periodic=True), c.p, ref_eqn(c.eqn))
    nx, ny = 512, 128
    yn = np.unique(c.mesh.nodes[:, 1])
    eqn = dataclasses.replace(c.eqn, wall_temperature=None)
    c = dataclasses.replace(c, mesh=mm.generate_channel(nx, ny, 4.0, yn, bottom="wall-adiabatic"), eqn=eqn)
    eid = lambda i, j: j * nx + i  # noqa: E731  (generate_channel's numbering)
    boundary = {(eid(i, 0), 0): "wall-adiabatic" for i in range(nx)}
    boundary.update({(eid(i, ny - 1), 2): "wall-slip" for i in range(nx)})
    pairs = [(eid(nx - 1, j), 1, eid(0, j), 3) for j in range(ny)]
    rm = rmesh.build_mesh(c.mesh.nodes, c.mesh.elements, boundary, pairs)
    return c, rsp.Discretization(rm, c.p, ref_eqn(c.eqn))


def rel(a, truth):
    return float(np.max(np.abs(np.asarray(a, dtype=np.longdouble) - truth)) / np.max(np.abs(truth)))


def main():
    out = {}
    for k in (2, 3, 4, 5):
        t0 = time.time()
        c, d = reference_case(k)
        tl = OracleDisc(c.mesh, c.p, c.eqn, dtype=np.longdouble)
        truth = tl.residual_mt(c.q0)
        rec = {"n_dofs": int(c.n_dofs), "max_abs_R": float(np.max(np.abs(truth)))}
        o = OracleDisc(c.mesh, c.p, c.eqn)
        rec["oracle_R_vs_truth"] = rel(o.residual_mt(c.q0), truth)
        if True:
            R0 = d.residual(c.q0)
            rec["reference_R_vs_truth"] = rel(R0, truth)
            if k == 2:
                X = np.random.default_rng(JV_SEED).uniform(-1.0, 1.0, c.n_dofs)
                qp = c.q0 + rnk.FD_EPS * X  # the reference's rounding of q + eps X
                Jt = JV_SHIFT * X.astype(np.longdouble) - (tl.residual_mt(qp) - truth) / rnk.FD_EPS
                rec["reference_Jv_vs_truth"] = rel(rnk.jfnk_matvec(X, c.q0, R0, d.residual, JV_SHIFT), Jt)
                rec["jv"] = {"shift": JV_SHIFT, "seed": JV_SEED, "eps": rnk.FD_EPS,
                             "max_abs_Jv": float(np.max(np.abs(Jt)))}
                del Jt, qp, X
            del R0
        del d, tl, truth, o
        gc.collect()
        rec["seconds"] = round(time.time() - t0, 1)
        out[f"config{k}"] = rec
        print(k, rec, flush=True)
    (HERE / "fullsize_floors.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
