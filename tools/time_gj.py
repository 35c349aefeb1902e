"""EJ block assembly + Gauss-Jordan inverse at config 2's fine level (p=4,
65,536 blocks of 100x100): CUDA-event time of assemble_element_blocks and a
digest of the factor (bitwise A/B of GJ tile shapes)."""
import hashlib, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2202_09733_b200 import cases, newton_krylov as nk
from paper_2202_09733_b200.spatial import Discretization
c = cases.config(2)
d = Discretization(c.mesh, c.p, c.eqn)
q = torch.as_tensor(c.q0, device="cuda")
B = nk.assemble_element_blocks(d, q, 5050.0, keep_blocks=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    B = nk.assemble_element_blocks(d, q, 5050.0, keep_blocks=False)
e1.record(); torch.cuda.synchronize()
print(f"assemble+invert {e0.elapsed_time(e1) / 3:.2f} ms  digest {hashlib.sha256(B.XT.cpu().numpy().tobytes()).hexdigest()[:16]}")
