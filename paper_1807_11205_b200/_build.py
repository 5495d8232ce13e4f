"""Build libgradsync_b200.so in-tree with nvcc for sm_100a.

The shared library is plain C ABI (include/gradsync_b200.h) with the CUDA
runtime linked statically, so it loads through ctypes next to torch without
any torch types crossing the boundary.  Output:
``paper_1807_11205_b200/_lib/libgradsync_b200.so``.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIBNAME = "libgradsync_b200.so"
LIBPATH = LIBDIR / LIBNAME

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # the bit-exact contract forbids contracting a*b+c into FFMA anywhere an
    # fp32 result is observable; explicit fma() calls (fp64 norms) are kept
    "-fmad=false",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
    "-I", str(ROOT / "include"),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libgradsync_b200")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _fingerprint() -> str:
    h = hashlib.sha256()
    for p in _sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "gradsync_b200.h"]:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every csrc/*.cu for sm_100a and link the shared library."""
    stamp = LIBDIR / ".fingerprint"
    fp = _fingerprint()
    if not force and LIBPATH.exists() and stamp.exists() and stamp.read_text() == fp:
        return LIBPATH
    LIBDIR.mkdir(exist_ok=True)
    objdir = LIBDIR / "obj"
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs, cmds = [], []
    for src in _sources():
        obj = objdir / (src.stem + ".o")
        cmds.append([nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
        objs.append(str(obj))
    # one nvcc per translation unit, concurrently (the LARS unit dominates)
    procs = []
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, pr in procs if pr.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    tmp = LIBDIR / (LIBNAME + ".tmp")
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
           "-cudart", "static", "-o", str(tmp), *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIBPATH)
    stamp.write_text(fp)
    return LIBPATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
