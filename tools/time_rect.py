"""A/B of the residual kernel families on the BASELINE configs: the
axis-aligned-rectangle path (csrc/fr_rect.cu) against the general bilinear
kernels (csrc/fr_kernels.cu).  CUDA-event times over rotating buffers
(>= 4x L2), R and fused Jv, plus the max relative difference of the two
paths' R.

    python tools/time_rect.py [configs...]      (default: 2 4; "2:p2" = config 2's mesh at degree 2)

"rect2" is the two-kernel chain (k_rgf + k_rasm), "rect4" the four-kernel
chain it replaced (k_rface + k_rgrad + k_rfc + k_rasm), "rect" the default
(the faster of the two per degree).  RECT_PATHS selects.
"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2202_09733_b200 import _lib, cases  # noqa: E402
from paper_2202_09733_b200.spatial import Discretization  # noqa: E402


def ev(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


import os
PATHS = tuple(os.environ.get("RECT_PATHS", "rect,rect4,general").split(","))


def main():
    ks = sys.argv[1:] or ["2", "4"]
    for arg in ks:
        k, _, pov = arg.partition(":p")
        k = int(k)
        c = cases.config(k)
        p = int(pov) if pov else c.p
        d = Discretization(c.mesh, p, c.eqn)
        if p != c.p:   # the same mesh and physics at another degree (a pMG level): perturbed free stream
            fs = d.free_stream_field().data.cpu().numpy().reshape(-1)
            c.q0 = fs * (1.0 + 0.01 * np.random.default_rng(0).standard_normal(fs.size))
        n = d.n_dofs
        nb = max(2, int(np.ceil(4 * 126e6 / (32.0 * n))))
        q0 = torch.as_tensor(c.q0, device="cuda")
        qs = [q0.clone() for _ in range(nb)]
        Rs = [torch.empty_like(q0) for _ in range(nb)]
        X = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
        R0 = d.residual(q0)
        reps = 10 if n > 1e8 else 100
        rec = {"config": k, "n_dofs": n, "p": p}
        outs = {}
        for path in PATHS:
            d.residual_path(path)
            r = lambda i: d.eval(qs[i % nb], _lib.EPI_R, Rs[i % nb])  # noqa: E731
            j = lambda i: d.eval(qs[i % nb], _lib.EPI_JV, Rs[i % nb], X=X, eps=1e-6, s=3.7, R0=R0)  # noqa: E731
            # the PTC matvec of a stage (X/dtau + (F(q + eps X) - Fk)/eps, three divisions per value)
            sj = lambda i: d.eval(qs[i % nb], _lib.EPI_STAGE_JV, Rs[i % nb], X=X, eps=1e-6, adt=0.0123, dtau=0.37,  # noqa: E731
                                  R0=R0, E=q0)
            df = lambda i: d.eval(qs[i % nb], _lib.EPI_DEFECT, Rs[i % nb], s=3.7, Sb=R0, Se=X)  # noqa: E731
            for i in range(3):
                r(i)
                j(i)
                sj(i)
                df(i)
            tr, tj, ts, td = ev(r, reps), ev(j, reps), ev(sj, reps), ev(df, reps)
            outs[path] = d.residual(q0).cpu().numpy()
            rec[path] = {"r_us": tr * 1e6, "r_gdofs": n / tr / 1e9, "jv_us": tj * 1e6, "jv_gdofs": n / tj / 1e9,
                         "stage_jv_us": ts * 1e6, "defect_us": td * 1e6}
        if "general" in outs:
            a, b = outs["rect"], outs["general"]
            rec["rect_vs_general"] = float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
            rec["speedup_r"] = rec["general"]["r_us"] / rec["rect"]["r_us"]
        if "rect4" in outs and "rect" in outs:
            rec["rect_bitwise_rect4"] = bool(np.array_equal(outs["rect"], outs["rect4"]))
        print(json.dumps(rec), flush=True)
        del d, qs, Rs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
