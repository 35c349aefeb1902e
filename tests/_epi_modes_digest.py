"""Helper for tests/test_gpu_residual.py: digests of every fused epilogue
mode's output at a small config-2 mesh (run in a subprocess so that
PMGB_EPI_SPECIALIZE is read fresh)."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2202_09733_b200 import _lib, cases  # noqa: E402
from paper_2202_09733_b200.spatial import Discretization  # noqa: E402

c = cases.config(2, nx=16)
rng = np.random.default_rng(11)
d4 = Discretization(c.mesh, c.p, c.eqn)
for d, q in ((d4, torch.as_tensor(c.q0, device="cuda")), (d4.coarsen(2), None)):
    if q is None:   # p=2 (the non-async assemble kernel): a restricted state
        from paper_2202_09733_b200 import pmg
        q = pmg._Transfer(d4, d).restrict(torch.as_tensor(c.q0, device="cuda"))
    n = q.numel()
    v = [torch.as_tensor(rng.standard_normal(n), device="cuda") for _ in range(4)]
    R0 = d.residual(q)
    outs = [
        d.eval(q, _lib.EPI_R),
        d.eval(q, _lib.EPI_F, s=3.5),
        d.eval(q, _lib.EPI_DEFECT, s=3.5, Sb=v[0], Se=v[1]),
        d.eval(q, _lib.EPI_JV, X=v[2], eps=1e-6, s=2.0, R0=R0),
        d.eval(q, _lib.EPI_STAGE_F, E=v[3], adt=0.3),
        d.eval(q, _lib.EPI_STAGE_JV, X=v[2], eps=1e-6, E=v[3], adt=0.3, dtau=0.7, R0=R0),
        d.eval(q, _lib.EPI_NEG_R),
        d.eval(q, _lib.EPI_OUTER_F, s=1.5, Se=v[1]),
    ]
    for o in outs:
        print(hashlib.sha256(o.cpu().numpy().tobytes()).hexdigest())
