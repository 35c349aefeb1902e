"""Exercise every hot kernel at BASELINE config 2 (for ncu / event timing).

    python tools/prof_kernels.py [reps]

Prints CUDA-event times per operation (warm, back to back)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2202_09733_b200 import _lib, cases, newton_krylov as nk, pmg  # noqa: E402
from paper_2202_09733_b200.spatial import Discretization  # noqa: E402
from paper_2202_09733_b200.vec import stream  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = cases.config(2)
d = Discretization(c.mesh, c.p, c.eqn)
q = torch.as_tensor(c.q0, device="cuda")
n = d.n_dofs
X = torch.randn(n, dtype=torch.float64, device="cuda")
R0 = d.residual(q)
out = torch.empty_like(q)


def timeit(name, fn, bytes_=None, flops=None):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    extra = ""
    if bytes_:
        extra += f"  {bytes_ / t / 1e9:8.1f} GB/s"
    if flops:
        extra += f"  {flops / t / 1e12:6.2f} TFLOP/s"
    print(f"{name:28s} {t * 1e6:10.1f} us  {n / t / 1e9:7.2f} GDoF/s{extra}", flush=True)
    return t


timeit("R", lambda: d.eval(q, _lib.EPI_R, out), flops=186.8 * n)
timeit("Jv", lambda: d.eval(q, _lib.EPI_JV, out, X=X, eps=1e-6, s=3.7, R0=R0))
timeit("defect", lambda: d.eval(q, _lib.EPI_DEFECT, out, s=3.7, Sb=R0, Se=X))
sz = d.elem_size
M = c.mesh.n_elements
invT = torch.empty((M, sz, sz), dtype=torch.float64, device="cuda")
perm = torch.empty((M, 2 * sz), dtype=torch.uint8, device="cuda")
lib = _lib.load()
t_asm = timeit("blocks assemble (fd only)",
               lambda: lib.pmgb_blocks_assemble(d._h, q.data_ptr(), 60.0, 1e-6, invT.data_ptr(), None, None,
                                                stream()))
t_inv = timeit("blocks invert (in place)",
               lambda: lib.pmgb_blocks_invert(M, sz, invT.data_ptr(), invT.data_ptr(), perm.data_ptr(), stream()),
               flops=2.0 * sz ** 3 * M)
lib.pmgb_blocks_assemble(d._h, q.data_ptr(), 60.0, 1e-6, invT.data_ptr(), invT.data_ptr(), perm.data_ptr(),
                         stream())
bj = nk.BlockJacobian(d, 60.0, invT, perm)
timeit("ej_update (block gemv)", lambda: bj.update(X, 1.0, q, out), bytes_=8.0 * (M * sz * sz + 3 * n))
ctx = pmg.PmgContext(d, pmg.PmgPrecondConfig(pmg.PHierarchy.parse("4-2", "2"), smoother_shift=50.0))
T = ctx.tables[0]
lo = T.restrict(q)
timeit("restrict 4->2", lambda: T.restrict(q, lo), bytes_=8.0 * (n + lo.numel()))
hi = q.clone()
timeit("prolong_add 2->4", lambda: T.prolong_add(lo, lo, hi), bytes_=8.0 * (2 * n + 2 * lo.numel()))
V = torch.randn((31, n), dtype=torch.float64, device="cuda")
Hd = torch.zeros(40, dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
w = X.clone()
timeit("mgs j=14", lambda: lib.pmgb_mgs(n, V.data_ptr(), n, 14, w.data_ptr(), Hd.data_ptr(), 0.0,
                                       flag.data_ptr(), stream()), bytes_=8.0 * n * (3 * 15 + 2))
