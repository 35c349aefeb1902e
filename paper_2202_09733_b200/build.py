"""Build libpmgflow_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2202_09733_b200.build [--verbose]

Each .cu is compiled to an object in parallel, then linked into one
shared library next to this file (it travels to the GPU box with the
repo snapshot; git ignores *.so).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libpmgflow_b200.so"
SOURCES = ["fr_kernels.cu", "fr_rect.cu", "fr_mixed.cu", "ej_kernels.cu", "krylov_kernels.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--fmad=true"]


def _compile(src: str, verbose: bool, defines=(), tag: str = "") -> Path:
    obj = CSRC / ("build" + tag) / (Path(src).stem + ".o")
    obj.parent.mkdir(exist_ok=True)
    cmd = [NVCC, *FLAGS, *defines, "-c", str(CSRC / src), "-o", str(obj)]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = obj.with_suffix(".log")
    log.write_text(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return obj


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [HERE.parent / "include" / "pmgflow_b200.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(verbose: bool = False, force: bool = False, defines=(), out: Path | None = None) -> Path:
    """Build the library; ``defines``/``out`` produce experiment variants
    (e.g. -DPMGB_CTA_THREADS=32 into libpmgflow_b200_v32.so) loaded via
    the PMGB_LIB environment variable -- the shipped default is LIB."""
    target = out or LIB
    if not force and out is None and not defines and not needs_build():
        return LIB
    tag = "" if target == LIB else "_" + target.stem
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, defines, tag), SOURCES))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(target),
           *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return target


if __name__ == "__main__":
    v = "--verbose" in sys.argv
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    out = HERE / outs[0] if outs else None
    print(build(verbose=v, force="--force" in sys.argv or v, defines=defs, out=out))
