"""EJ block apply at config 2's fine level (p=4, 65,536 blocks of 100x100):
FP64-stored vs FP32-stored factor, CUDA-event time and the stream's
algorithmic bytes (factor + perm + x gather + y) per apply.
    python tools/time_ej.py [nx] [reps]"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, newton_krylov as nk
from paper_2202_09733_b200.spatial import Discretization

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = cases.config(2, nx=nx)
d = Discretization(c.mesh, c.p, c.eqn)
q = torch.as_tensor(c.q0, device="cuda")
M, sz = c.mesh.n_elements, d.elem_size
X = torch.randn(d.n_dofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
out = {"M": M, "sz": sz}
for prec in ("fp64", "fp32"):
    B = nk.assemble_element_blocks(d, q, 5000.0 + 50.0, keep_blocks=False, precision=prec)
    y = B.apply(X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        B.apply(X)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    nbytes = M * sz * sz * B.XT.element_size() + M * 2 * sz + 2 * 8 * M * sz
    out[prec] = {"us": t * 1e6, "GBps": nbytes / t / 1e9, "bytes": nbytes}
    if prec == "fp64":
        y64 = y.clone()
    else:
        out["rel_diff_fp32_vs_fp64"] = float((y - y64).abs().max() / y64.abs().max())
    del B
    torch.cuda.empty_cache()
print(json.dumps(out))
