"""Pinned host<->device copy bandwidth for a 52 MB vector: H2D, D2H, and
both at once on two streams (the e2e path's ceiling)."""
import torch
n = 6553600
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3
def h2d():
    d_a.copy_(h_in, non_blocking=True)
def d2h():
    h_out.copy_(d_b, non_blocking=True)
def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
B = 8 * n
for name, fn in (("H2D", h2d), ("D2H", d2h), ("H2D+D2H concurrent", both)):
    t = timeit(fn)
    print(f"{name}: {t*1e3:.3f} ms per 52 MB each way -> {B/t/1e9:.1f} GB/s per direction", flush=True)
