"""Compile the CUDA sources into the in-tree C-ABI library (sm_100a only).

    python -m paper_2408_01331_b200.build_lib      # or __graft_entry__.build()

Produces paper_2408_01331_b200/_lib/libhnn_b200.so with plain nvcc (no torch
extension machinery): extern "C" entry points declared in include/hnn_b200.h.
Objects are rebuilt only when a source or header is newer than the library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libhnn_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
PER_FILE_FLAGS: dict = {}
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    return "nvcc"


def sources() -> list:
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps: list) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False) -> Path:
    OUT_DIR.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [REPO / "include" / "hnn_b200.h"]
    objs = []
    log = []
    for src in sources():
        obj = OUT_DIR / (src.stem + ".o")
        objs.append(obj)
        if _stale(obj, [src] + headers):
            extra = PER_FILE_FLAGS.get(src.name, [])
            cmd = [_nvcc(), *ARCH, *FLAGS, *extra, "-I", str(REPO / "include"), "-c", str(src), "-o", str(obj)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            log.append(r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stderr)
                raise RuntimeError(f"nvcc failed on {src.name}")
    if _stale(LIB, objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stderr)
            raise RuntimeError("nvcc link failed")
    if verbose:
        sys.stderr.write("".join(log))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
