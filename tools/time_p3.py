"""R at p=3 on 65536 elements: periodic box (config-1 physics at nx=256)
vs the config-4 channel -- separates degree from walls/stretching."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, _lib
from paper_2202_09733_b200.spatial import Discretization
for name, c in (("config1@256 (periodic box, p3)", cases.config(1, nx=256)), ("config4 (channel, p3)", cases.config(4)),
                ("config2@128 (periodic box, p4)", cases.config(2, nx=128))):
    d = Discretization(c.mesh, c.p, c.eqn)
    qs = [torch.as_tensor(c.q0, device="cuda") for _ in range(4)]
    out = torch.empty_like(qs[0])
    for i in range(3):
        d.eval(qs[i % 4], _lib.EPI_R, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(40):
        d.eval(qs[i % 4], _lib.EPI_R, out)
    e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1) / 40 * 1e-3
    print(f"{name}: {t*1e6:.1f} us, {d.n_dofs/t/1e9:.2f} GDoF/s ({d.n_dofs} DoF)", flush=True)
