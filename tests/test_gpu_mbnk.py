"""Device MBNK path through the C ABI against the reference's goldens
(tests/golden/make_golden_mbnk.py) and the oracle: block-sparse FD
Jacobian (element + coupling blocks), block SpMV, block ILU0 factor and
apply, MBNK-smoothed pMG, switch_after.  FD blocks carry the reference's
own FD noise (R rounding x 1/eps), hence ~1e-7-of-scale tolerances."""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2202_09733_b200 import cases, mesh as mm, newton_krylov as nk
from paper_2202_09733_b200.equation import EquationSpec
from paper_2202_09733_b200.spatial import Discretization

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).parent / "golden" / "golden_mbnk.npz")

SPARSE_CASES = {
    "box3p_ns1": (lambda: mm.generate_box(3, 3, 1.0, 1.0, periodic=True),
                  dict(kind="navier-stokes", mach=0.3, reynolds=100.0), 1),
    "box2p_ns1": (lambda: mm.generate_box(2, 2, 1.0, 1.0, periodic=True),
                  dict(kind="navier-stokes", mach=0.3, reynolds=100.0), 1),
    "cyl_ns1": (lambda: mm.generate_cylinder_omesh(12, 4, 0.5, 8.0, 1.3),
                dict(kind="navier-stokes", mach=0.3, reynolds=200.0), 1),
    "box3ff_euler2": (lambda: mm.generate_box(3, 3, 2.0, 1.5), dict(kind="euler", mach=0.3), 2),
}


def scaled(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def t(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


@pytest.mark.parametrize("name", list(SPARSE_CASES))
def test_sparse_blocks_match_reference(cuda, name):
    mk, kw, p = SPARSE_CASES[name]
    d = Discretization(mk(), p, EquationSpec(**kw))
    pre = f"sp/{name}/"
    A = nk.assemble_sparse_blocks(d, t(G[pre + "q"]), 40.0)
    assert np.array_equal(A.indptr, G[pre + "indptr"]) and np.array_equal(A.indices, G[pre + "indices"])
    assert scaled(A.blocks, G[pre + "blocks"]) <= 1e-7
    assert scaled(A.matvec(t(G[pre + "X"])), G[pre + "AX"]) <= 1e-7
