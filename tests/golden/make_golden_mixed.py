"""Golden vectors of the REFERENCE on mixed-degree meshes.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_mixed.py

The reference's Discretization with a per-element degree map
(spatial.py:295-359): degree groups, mortar faces (_pair_align /
_pair_scatter, 468-497, 572-585).  For a periodic box, a far-field box, a
stretched (non-rectangular-free) channel with walls and a curved O-grid,
Euler and Navier-Stokes: R(q) (501-570), the frozen neighbour records of
freeze (700-766; q, w and fvn per interior element face, zero-padded to 6
points) and element_residual (768-853) of a few elements for a batch of
perturbed states.  Also p_adapt.nest_hierarchy (106-123) over a table of
inputs and one adapt event (71-103).  Output: golden_mixed.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from pmgflow import mesh as rmesh  # noqa: E402
from pmgflow import p_adapt as rpa  # noqa: E402
from pmgflow import spatial as rsp  # noqa: E402


def meshes():
    yn = np.array([0.0, 0.03, 0.1, 0.25, 0.5, 1.0])
    nx = 5
    X, Y = np.meshgrid(np.linspace(0.0, 2.0, nx + 1), yn)
    nodes = np.stack([X.ravel(), Y.ravel()], axis=1)
    jj, ii = np.meshgrid(np.arange(5), np.arange(nx), indexing="ij")
    base = (jj * (nx + 1) + ii).ravel()
    elements = np.stack([base, base + 1, base + nx + 2, base + nx + 1], axis=1)
    eid = lambda i, j: j * nx + i  # noqa: E731
    bnd = {(eid(i, 0), 0): "wall-adiabatic" for i in range(nx)}
    bnd.update({(eid(i, 4), 2): "wall-slip" for i in range(nx)})
    chan = rmesh.build_mesh(nodes, elements, bnd, [(eid(nx - 1, j), 1, eid(0, j), 3) for j in range(5)])
    return {
        "boxp": rmesh.generate_box(5, 4, 2.0, 1.5, periodic=True),
        "boxff": rmesh.generate_box(4, 4, 2.0, 2.0),
        "chan": chan,
        "cyl": rmesh.generate_cylinder_omesh(12, 3, 0.5, 6.0, 1.3),
    }


def degree_map(m, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(1, 5, m.n_elements)


def main():
    out = {}
    kinds = {"euler": dict(kind="euler", mach=0.3), "ns": dict(kind="navier-stokes", mach=0.3, reynolds=150.0)}
    for mi, (mname, m) in enumerate(meshes().items()):
        deg = degree_map(m, 10 + mi)
        deg[0], deg[1] = 0 if mname == "boxff" else deg[0], 5 if mname == "boxp" else deg[1]
        for kname, kw in kinds.items():
            d = rsp.Discretization(m, deg, rsp.EquationSpec(**kw))
            rng = np.random.default_rng(7 + mi)
            q = d.free_stream_field().data * (1 + 0.02 * rng.standard_normal(d.n_dofs))
            key = f"{mname}/{kname}"
            out[f"{key}/degrees"] = deg
            out[f"{key}/q"] = q
            out[f"{key}/R"] = d.residual(q)
            fr = d.freeze(q)
            M = m.n_elements
            rq = np.zeros((M, 4, 6, 4))
            rw = np.zeros((M, 4, 6, 3))
            rf = np.zeros((M, 4, 6, 4))
            for e in range(M):
                for f in range(4):
                    rec = fr[e][f]
                    if rec[0] != "interior":
                        continue
                    n = len(rec[2]["q"])
                    rq[e, f, :n] = rec[2]["q"]
                    if "w" in rec[2]:
                        rw[e, f, :n] = rec[2]["w"]
                        rf[e, f, :n] = rec[2]["fvn"]
            out[f"{key}/rq"], out[f"{key}/rw"], out[f"{key}/rf"] = rq, rw, rf
            for e in (0, 1, M - 1):
                n = int(deg[e]) + 1
                Q = q[d.offsets[e]:d.offsets[e + 1]].reshape(n, n, 4)
                B = np.stack([Q, Q * 1.001, Q * (1 + 0.003 * rng.standard_normal(Q.shape))])
                out[f"{key}/local/e{e}/Q"] = B
                out[f"{key}/local/e{e}/R"] = d.element_residual(e, B, fr)
    tab = []
    for levels in ((4, 2), (4, 3, 2, 1, 0), (5, 4), (3, 2, 1)):
        for p_e in range(levels[0] + 1):
            tab.append(list(rpa.nest_hierarchy(p_e, levels[0], levels)) + [-1] * (5 - len(levels)))
    out["nest/table"] = np.array(tab)
    m = rmesh.generate_box(4, 4, 2.0, 2.0, periodic=True)
    d = rsp.Discretization(m, 3, rsp.EquationSpec(kind="euler", mach=0.3))
    xy = d.groups[0].xy
    q = d.free_stream_field()
    bump = np.exp(-((xy[..., 0] - 1.0) ** 2 + (xy[..., 1] - 1.0) ** 2) / 0.05)
    Q = q.data.reshape(-1, 4, 4, 4).copy()
    Q[..., 1] *= 1.0 + 0.5 * bump
    q.data[:] = Q.reshape(-1)
    cfg = rpa.AdaptConfig(variable="momentum-x", nu_max=0.2, nu_min=0.001, p_min=1, p_max=4)
    new, eta = rpa.adapt(q, cfg)
    out["adapt/q"], out["adapt/eta"] = q.data.copy(), eta
    out["adapt/degrees"], out["adapt/q_new"] = new.degrees, new.data
    np.savez_compressed(HERE / "golden_mixed.npz", **out)
    print({k: v.shape for k, v in out.items() if k.endswith("/R")})


if __name__ == "__main__":
    main()
