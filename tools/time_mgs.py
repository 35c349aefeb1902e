"""MGS Arnoldi step at config-2 size (6.55 M DoF): pmgb_mgs for j = 0..29
(one GMRES(30) cycle's orthogonalisations), CUDA-event time and the
algorithmic bytes (32 B/DoF per projection pass + the norm and normalise)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200._lib import check, load
from paper_2202_09733_b200.vec import ptr, stream

n = 6553600
m = 30
g = torch.Generator("cuda").manual_seed(1)
V = torch.randn((m + 1, n), dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
H = torch.zeros((m, m + 2), dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
W = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
lib = load()
def cycle():
    for j in range(m):
        w = W[j].clone()
        check(lib.pmgb_mgs(n, V.data_ptr(), n, j, ptr(w), H[j].data_ptr(), 0.0, flag.data_ptr(), stream()), "mgs")
for _ in range(2):
    cycle()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); cycle(); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e-3
passes = sum(j + 2 for j in range(m))
alg = passes * 32.0 * n
print(json.dumps({"cycle_ms": t * 1e3, "passes": passes, "alg_GBps": alg / t / 1e9,
                  "h_checksum": float(H.sum().item())}))
