"""Golden wall forces (compute_forces, spatial.py:633-695), made by running
the REFERENCE pmgflow in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_forces.py

Cylinder O-mesh with adiabatic (NS) and slip (Euler) walls at p=2, and the
reduced config-4 channel (adiabatic bottom wall, slip top) at p=3.
Written to tests/golden/golden_forces.npz."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

from pmgflow import mesh as rmesh  # noqa: E402
from pmgflow import spatial as rsp  # noqa: E402

from paper_2202_09733_b200 import cases  # noqa: E402


def main():
    out = {}
    for name, m, kw, p in (
            ("cyl_ns2", rmesh.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3),
             dict(kind="navier-stokes", mach=0.3, reynolds=200.0), 2),
            ("cyl_slip_euler2", rmesh.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3, wall_tag="wall-slip"),
             dict(kind="euler", mach=0.3), 2)):
        d = rsp.Discretization(m, p, rsp.EquationSpec(**kw))
        rng = np.random.default_rng(5)
        q = d.free_stream_field().data * (1 + 0.02 * rng.standard_normal(d.n_dofs))
        out[f"{name}/q"] = q
        out[f"{name}/F"] = np.array(d.compute_forces(q))
    c = cases.config(4, nx=16)
    e = c.eqn
    eqn = rsp.EquationSpec(kind=e.kind, mach=e.mach, reynolds=e.reynolds, ref_length=e.ref_length)
    from pmgflow.mesh import build_mesh  # noqa: F401  (the channel comes from the same node arrays)
    m = rmesh.Mesh(nodes=c.mesh.nodes, elements=c.mesh.elements, interior_faces=c.mesh.interior_faces,
                   boundary_faces=c.mesh.boundary_faces, boundary_tags=list(c.mesh.boundary_tags))
    d = rsp.Discretization(m, 3, eqn)
    out["chan_ns3/q"] = c.q0
    out["chan_ns3/F"] = np.array(d.compute_forces(c.q0))
    np.savez_compressed(HERE / "golden_forces.npz", **out)
    print({k: v for k, v in out.items() if k.endswith("/F")})


if __name__ == "__main__":
    main()
