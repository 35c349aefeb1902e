"""The C ABI library loads and exports every symbol include/pmgflow_b200.h
declares (no compute calls: runs on the CPU-only build box)."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pmgflow_b200.h"


def declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"PMGB_API\s+[\w\s\*]+?\b(pmgb_\w+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    assert "pmgb_residual" in names and "pmgb_mgs" in names and len(names) >= 25


def test_library_exports_all_declared_symbols():
    from paper_2202_09733_b200 import _lib, build
    if build.needs_build():
        build.build()
    lib = _lib.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    # the binding declares exactly the header's symbols
    assert sorted(_lib.SIGNATURES) == declared()


def test_version_string_without_gpu():
    from paper_2202_09733_b200 import _lib
    assert b"sm_100a" in _lib.load().pmgb_version()
