"""R / defect / PTC-Jv at config 2's coarse level (p=2, 65,536 elements)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, _lib, pmg
from paper_2202_09733_b200.spatial import Discretization
c = cases.config(2)
d4 = Discretization(c.mesh, 4, c.eqn)
d = d4.coarsen(2)
q = pmg._Transfer(d4, d).restrict(torch.as_tensor(c.q0, device="cuda"))
X = torch.randn_like(q); Sb = torch.randn_like(q); Se = torch.randn_like(q)
R0 = d.residual(q)
res = []
for name, kw in (("R", dict(mode=_lib.EPI_R)), ("defect", dict(mode=_lib.EPI_DEFECT, s=3.0, Sb=Sb, Se=Se)),
                 ("stage_jv", dict(mode=_lib.EPI_STAGE_JV, X=X, eps=1e-6, E=Sb, adt=0.3, dtau=0.5, R0=R0))):
    mode = kw.pop("mode")
    for _ in range(3):
        d.eval(q, mode, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        d.eval(q, mode, **kw)
    e1.record(); torch.cuda.synchronize()
    res.append(f"{name} {e0.elapsed_time(e1) * 10:.1f} us")
print(" | ".join(res))
