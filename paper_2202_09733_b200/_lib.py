"""ctypes binding of libpmgflow_b200.so (the C ABI in include/pmgflow_b200.h).

This is the reference-side binding a maintainer would add to pmgflow
(INTEGRATION.md shows it next to each replaced call site).  There is no
CPU fallback: if the shared library is missing or no CUDA device is
present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_LIB_PATH = Path(os.environ.get("PMGB_LIB") or Path(__file__).resolve().with_name("libpmgflow_b200.so"))
_lib = None

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_void_p = ctypes.c_void_p


class DiscDesc(ctypes.Structure):
    _fields_ = [
        ("n_elem", ctypes.c_int64), ("degree", ctypes.c_int32), ("kind", ctypes.c_int32),
        ("gamma", ctypes.c_double), ("mu", ctypes.c_double), ("kappa", ctypes.c_double),
        ("adv_x", ctypes.c_double), ("adv_y", ctypes.c_double), ("diffusivity", ctypes.c_double),
        ("free_stream", c_double_p), ("D", c_double_p), ("eL", c_double_p), ("eR", c_double_p),
        ("lL", c_double_p), ("lR", c_double_p), ("xg", c_double_p), ("geom", c_double_p),
        ("links", c_int64_p), ("tags", c_int32_p),
        ("riemann", ctypes.c_int32), ("viscous_scheme", ctypes.c_int32),
        ("wall_temperature", ctypes.c_double),
    ]


class Epilogue(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("s", ctypes.c_double), ("eps", ctypes.c_double), ("adt", ctypes.c_double),
        ("dtau", ctypes.c_double), ("sb_scalar", ctypes.c_double), ("se_scalar", ctypes.c_double),
        ("X", c_void_p), ("R0", c_void_p), ("E", c_void_p), ("Sb", c_void_p), ("Se", c_void_p),
        ("Q0", c_void_p), ("dtau_e", c_void_p), ("alpha", ctypes.c_double),
    ]


EPI_R, EPI_F, EPI_DEFECT, EPI_JV, EPI_STAGE_F, EPI_STAGE_JV, EPI_NEG_R, EPI_OUTER_F, EPI_RK = range(9)

# name -> (restype, argtypes); exactly the symbols include/pmgflow_b200.h declares
SIGNATURES = {
    "pmgb_disc_create": (ctypes.c_int, [ctypes.POINTER(DiscDesc), ctypes.POINTER(c_void_p)]),
    "pmgb_disc_destroy": (ctypes.c_int, [c_void_p]),
    "pmgb_disc_n_dofs": (ctypes.c_int64, [c_void_p]),
    "pmgb_disc_residual_path": (ctypes.c_int, [c_void_p, ctypes.c_int32]),
    "pmgb_mdisc_create": (ctypes.c_int, [ctypes.POINTER(DiscDesc), c_int32_p, c_double_p, c_double_p,
                                         ctypes.POINTER(c_void_p)]),
    "pmgb_mdisc_destroy": (ctypes.c_int, [c_void_p]),
    "pmgb_mdisc_n_dofs": (ctypes.c_int64, [c_void_p]),
    "pmgb_mdisc_eval": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, ctypes.c_double, ctypes.POINTER(Epilogue),
                                       c_void_p, c_void_p]),
    "pmgb_mdisc_freeze": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_mdisc_element_residual": (ctypes.c_int, [c_void_p, ctypes.c_int32, c_void_p, ctypes.c_int64, c_void_p,
                                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_residual": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_rk_lambda": (ctypes.c_int, [c_void_p, c_void_p, ctypes.c_double, c_void_p, c_void_p]),
    "pmgb_rk_dtau": (ctypes.c_int, [ctypes.c_int64, c_void_p, ctypes.c_double, ctypes.c_double, c_void_p,
                                    c_void_p]),
    "pmgb_eval": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, ctypes.c_double,
                                 ctypes.POINTER(Epilogue), c_void_p, c_void_p]),
    "pmgb_jfnk_matvec": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, ctypes.c_double,
                                        ctypes.c_double, c_void_p, c_void_p]),
    "pmgb_freeze": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_element_residual": (ctypes.c_int, [c_void_p, c_void_p, ctypes.c_int64, c_void_p, c_void_p,
                                             c_void_p, c_void_p, c_void_p]),
    "pmgb_blocks_assemble": (ctypes.c_int, [c_void_p, c_void_p, ctypes.c_double, ctypes.c_double,
                                            c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_blocks_invert": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_sparse_matvec": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_void_p]),
    "pmgb_ilu0_factor": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_ilu0_apply": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p, ctypes.c_int32, c_void_p, c_void_p, ctypes.c_int32, c_void_p,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_wall_forces": (ctypes.c_int, [c_void_p, c_void_p, ctypes.c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p]),
    "pmgb_ilu0_apply_fused": (ctypes.c_int, [ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                             ctypes.c_int32, c_void_p, c_void_p, ctypes.c_int32, c_void_p, c_void_p,
                                             ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_sparse_assemble": (ctypes.c_int, [c_void_p, c_void_p, ctypes.c_double, ctypes.c_double, c_void_p,
                                            c_void_p, ctypes.c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_void_p, ctypes.c_int32, c_void_p]),
    "pmgb_ej_apply": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_void_p]),
    "pmgb_ej_update": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p,
                                      ctypes.c_double, c_void_p, c_void_p, c_void_p]),
    "pmgb_blocks_demote": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p]),
    "pmgb_ej_apply_f32": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p]),
    "pmgb_ej_update_f32": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p, c_void_p,
                                          ctypes.c_double, c_void_p, c_void_p, c_void_p]),
    "pmgb_transfer": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     c_double_p, c_void_p, c_void_p, c_void_p, ctypes.c_int32, c_void_p]),
    "pmgb_dot": (ctypes.c_int, [ctypes.c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pmgb_nrm2": (ctypes.c_int, [ctypes.c_int64, c_void_p, c_void_p, c_void_p]),
    "pmgb_mgs_pass": (ctypes.c_int, [ctypes.c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                     ctypes.c_int32, c_void_p, c_void_p]),
    "pmgb_normalize_sqrt": (ctypes.c_int, [ctypes.c_int64, c_void_p, c_void_p, ctypes.c_double, c_void_p,
                                           c_void_p]),
    "pmgb_mgs": (ctypes.c_int, [ctypes.c_int64, c_void_p, ctypes.c_int64, ctypes.c_int32, c_void_p,
                                c_void_p, ctypes.c_double, c_void_p, c_void_p]),
    "pmgb_lincomb": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_double_p,
                                    ctypes.POINTER(c_void_p), c_void_p, c_void_p]),
    "pmgb_gemv_t": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, ctypes.c_int64, c_void_p,
                                   c_void_p, c_void_p]),
    "pmgb_any_nonzero": (ctypes.c_int, [ctypes.c_int64, c_void_p, c_void_p, c_void_p]),
    "pmgb_multidot": (ctypes.c_int, [ctypes.c_int64, c_void_p, ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p,
                                     c_void_p, c_void_p]),
    "pmgb_gemv_sub": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, ctypes.c_int64, c_void_p, c_void_p,
                                     c_void_p]),
    "pmgb_status": (ctypes.c_int, [c_void_p, c_int32_p, c_int64_p, ctypes.c_int32]),
    "pmgb_status_clear": (ctypes.c_int, [c_void_p]),
    "pmgb_sync": (ctypes.c_int, [c_void_p]),
    "pmgb_error_string": (ctypes.c_char_p, [ctypes.c_int]),
    "pmgb_version": (ctypes.c_char_p, []),
    "pmgb_probe_fp64": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, c_void_p, c_void_p]),
    "pmgb_launch_count": (ctypes.c_int64, []),
}


class PmgbError(RuntimeError):
    pass


def lib_path() -> Path:
    return _LIB_PATH


def load():
    """Load the shared library and declare every exported symbol."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"{_LIB_PATH.name} is not built; run "
                              "`python -m paper_2202_09733_b200.build` (nvcc, sm_100a)")
        lib = ctypes.CDLL(str(_LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = load().pmgb_error_string(int(rc)).decode()
        raise PmgbError(f"{what}: pmgflow_b200 error {rc}: {msg}")
