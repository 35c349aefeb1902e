"""pMG transfers at config 2 (p4 <-> p2, 65,536 elements): restriction and
prolong-add, CUDA-event time, HBM bytes, and a digest for bitwise A/B."""
import hashlib, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, pmg
from paper_2202_09733_b200.spatial import Discretization

c = cases.config(2)
d4 = Discretization(c.mesh, 4, c.eqn)
d2 = d4.coarsen(2)
tr = pmg._Transfer(d4, d2)
q = torch.as_tensor(c.q0, device="cuda")
qc = tr.restrict(q)
base = qc * 0.999
out = {}
for name, fn, nbytes in (("restrict", lambda: tr.restrict(q), 8 * (q.numel() + qc.numel())),
                         ("prolong_add", lambda: tr.prolong_add(qc, base, q.clone()), 8 * (3 * q.numel() + 2 * qc.numel()))):
    for _ in range(3):
        r = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 50 * 1e-3
    out[name] = {"us": round(t * 1e6, 1), "digest": hashlib.sha256(r.cpu().numpy().tobytes()).hexdigest()[:16]}
print(json.dumps(out))
