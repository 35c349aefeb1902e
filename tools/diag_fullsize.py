import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2202_09733_b200 import cases
from paper_2202_09733_b200.spatial import Discretization
for k in [int(a) for a in sys.argv[1:]]:
    t = time.time(); c = cases.config(k); print("build", k, time.time() - t, flush=True)
    d = Discretization(c.mesh, c.p, c.eqn)
    fs = d.free_stream_field().data
    R = d.residual(fs)
    a = R.abs().reshape(c.mesh.n_elements, -1)
    em = a.max(1).values
    print("fs max", float(a.max()), "n bad elems", int((em > 1e-11).sum()), "first", torch.nonzero(em > 1e-11)[:5].flatten().tolist(), flush=True)
    fsn = fs.cpu().numpy().reshape(-1, 4)
    print("fs state", fsn[0], "spread", fsn.max(0) - fsn.min(0))
    q = torch.as_tensor(c.q0, device="cuda")
    R = d.residual(q)
    fr = d.freeze(q)
    M = c.mesh.n_elements
    elems = np.arange(0, M, max(1, M // 64))
    sz = d.elem_size
    Q = torch.stack([q[e * sz:(e + 1) * sz] for e in elems]).reshape(len(elems), d.n, d.n, d.nvars)
    Rl = d.element_residual(elems, Q, fr).reshape(len(elems), sz)
    Rg = torch.stack([R[e * sz:(e + 1) * sz] for e in elems])
    print("local-global", float((Rl - Rg).abs().max()), "Rmax", float(R.abs().max()),
          "per-elem rel", float(((Rl - Rg).abs().max(1).values / Rg.abs().max(1).values).max()), flush=True)
