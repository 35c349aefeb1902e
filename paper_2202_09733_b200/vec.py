"""Device vectors: FP64 CUDA tensors plus the library's BLAS-1 kernels.

PyTorch provides the allocations and the current stream; every
arithmetic kernel on the solver path is a libpmgflow_b200 launch.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import check, load

_scratch = {}

# Element-partitioned solves (paper_2202_09733_b200.partition): while a
# partition is active, every reduction on the solver path (nrm2, dot,
# any_nonzero, the GMRES Arnoldi step, the status word) runs over the
# rank's OWNED elements and is summed / max-ed over the ranks; the halo
# entries of a strip vector are never reduced.
_PART = None


def set_partition(part):
    """Activate (or, with None, clear) the partition reductions use."""
    global _PART
    _PART = part


def active_partition():
    return _PART


def owned(x: torch.Tensor) -> torch.Tensor:
    """The owned-element range of an element-major strip vector (any level:
    the per-element size is x.numel() / n_local)."""
    if _PART is None:
        return x
    sz = x.numel() // _PART.n_local
    return x[_PART.owned.start * sz:_PART.owned.stop * sz]


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2202_09733_b200 needs a CUDA device (sm_100a); no CPU fallback")


def ptr(t: torch.Tensor) -> int:
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("expected a contiguous float64 CUDA tensor")
    return t.data_ptr()


def to_device(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == torch.float64 and x.is_contiguous():
            return x
        return x.to(device=device or "cuda", dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to(device or "cuda")


def _scalars(device, n=4):
    key = (str(device), n)
    t = _scratch.get(key)
    if t is None:
        t = torch.zeros(n, dtype=torch.float64, device=device)
        _scratch[key] = t
    return t


def lincomb(coeffs, xs, out=None) -> torch.Tensor:
    """out = sum c_i x_i (k <= 8), one fused kernel."""
    k = len(xs)
    if k == 0 or k > 8:
        raise ValueError("lincomb takes 1..8 vectors")
    n = xs[0].numel()
    if out is None:
        out = torch.empty_like(xs[0])
    c = (ctypes.c_double * k)(*[float(v) for v in coeffs])
    p = (ctypes.c_void_p * k)(*[ptr(x) for x in xs])
    check(load().pmgb_lincomb(n, k, c, p, ptr(out), stream()), "lincomb")
    return out


def axpby(a, x, b, y, out=None):
    return lincomb((a, b), (x, y), out)


def nrm2_dev(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=x.device)
    check(load().pmgb_nrm2(x.numel(), ptr(x), out.data_ptr(), stream()), "nrm2")
    return out


def nrm2(x: torch.Tensor) -> float:
    """||x||_2 = sqrt(x . x) with a fixed-order reduction (synchronising);
    partitioned: sqrt of the rank-summed owned x . x."""
    if _PART is not None:
        return float(np.sqrt(dot(x, x)))
    s = _scalars(x.device)
    nrm2_dev(x, s[0:1])
    return float(s[0].item())


def dot(x: torch.Tensor, y: torch.Tensor) -> float:
    s = _scalars(x.device)
    if _PART is not None:
        xo, yo = owned(x), owned(y)
        check(load().pmgb_dot(xo.numel(), ptr(xo), ptr(yo), s.data_ptr(), stream()), "dot")
        return _PART.allreduce(float(s[0].item()), "sum")
    check(load().pmgb_dot(x.numel(), ptr(x), ptr(y), s.data_ptr(), stream()), "dot")
    return float(s[0].item())


def any_nonzero(x: torch.Tensor) -> bool:
    f = torch.zeros(1, dtype=torch.int32, device=x.device)
    xo = owned(x)
    check(load().pmgb_any_nonzero(xo.numel(), ptr(xo), f.data_ptr(), stream()), "any_nonzero")
    if _PART is not None:
        return _PART.allreduce(float(f.item()), "max") > 0.0
    return bool(f.item())


def launch_count() -> int:
    return int(load().pmgb_launch_count())
