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


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: tuple = (), only: tuple = ()) -> Path:
    """Compile every csrc/*.cu for sm_100a and link the shared library.

    variant/defines: a tuning build (extra -D flags) linked to
    _lib/variants/libgradsync_b200_<variant>.so for A/B measurements (load
    it with GRADSYNC_B200_LIB); the product library is untouched.  only:
    translation units (stems) a variant recompiles; the others are the
    product build's objects."""
    libdir = LIBDIR / "variants" if variant else LIBDIR
    libpath = libdir / (f"libgradsync_b200_{variant}.so" if variant else LIBNAME)
    flags = NVCC_FLAGS + [f"-D{d}" for d in defines]
    stamp = libdir / (f".fingerprint_{variant}" if variant else ".fingerprint")
    fp = _fingerprint() + " ".join(defines)
    if not force and libpath.exists() and stamp.exists() and stamp.read_text() == fp:
        return libpath
    libdir.mkdir(parents=True, exist_ok=True)
    objdir = libdir / (f"obj_{variant}" if variant else "obj")
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs, cmds = [], []
    for src in _sources():
        if variant and only and src.stem not in only:
            objs.append(str(LIBDIR / "obj" / (src.stem + ".o")))  # the product build's
            continue
        obj = objdir / (src.stem + ".o")
        cmds.append([nvcc, *flags, "-c", str(src), "-o", str(obj)])
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
    tmp = libdir / (libpath.name + ".tmp")
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
           "-cudart", "static", "-o", str(tmp), *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, libpath)
    stamp.write_text(fp)
    return libpath


if __name__ == "__main__":
    # python -m paper_1807_11205_b200._build [--force] [--variant NAME -DMACRO=V ...]
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    only = tuple(args[args.index("--only") + 1].split(",")) if "--only" in args else ()
    if var and only:
        build()  # the product objects the variant links against
    print(build(force="--force" in args, verbose=True, variant=var, defines=defs, only=only))
