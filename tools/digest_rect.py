"""SHA-256 digests of R, Jv, the stage-Jv and the defect form on the rectangle
path (two- and four-kernel chains) for an experiment build (PMGB_LIB=...):
two builds whose digests agree are bitwise equal on these cases.

    PMGB_LIB=... python tools/digest_rect.py [configs...]   (default 2 4; reduced meshes, "k:nx")
"""
import hashlib
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2202_09733_b200 import _lib, cases  # noqa: E402
from paper_2202_09733_b200.spatial import Discretization  # noqa: E402


def dig(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]


for arg in sys.argv[1:] or ["2", "4"]:
    k, _, nx = arg.partition(":")
    c = cases.config(int(k), nx=int(nx)) if nx else cases.config(int(k))
    d = Discretization(c.mesh, c.p, c.eqn)
    q0 = torch.as_tensor(c.q0, device="cuda")
    X = torch.randn(d.n_dofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
    rec = {"config": arg, "n_dofs": d.n_dofs}
    for path in ("rect2", "rect4"):
        d.residual_path(path)
        R0 = d.residual(q0)
        out = torch.empty_like(q0)
        rec[path] = {"R": dig(R0),
                     "Jv": dig(d.eval(q0, _lib.EPI_JV, out, X=X, eps=1e-6, s=3.7, R0=R0)),
                     "stageJv": dig(d.eval(q0, _lib.EPI_STAGE_JV, out, X=X, eps=1e-6, adt=0.0123, dtau=0.37, R0=R0,
                                           E=q0)),
                     "defect": dig(d.eval(q0, _lib.EPI_DEFECT, out, s=3.7, Sb=R0, Se=X))}
    print(json.dumps(rec), flush=True)
