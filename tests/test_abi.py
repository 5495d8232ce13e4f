"""The C-ABI library loads and exports every symbol include/gradsync_b200.h
declares, with the struct layouts the Python side assumes (CPU: no kernel is
launched here)."""

import ctypes
import re
from pathlib import Path

import numpy as np

from paper_1807_11205_b200 import _build, _native

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    text = (ROOT / "include" / "gradsync_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", text)))


def test_library_built_for_sm100a():
    _build.build()
    assert _build.LIBPATH.exists()
    assert "arch=compute_100a,code=sm_100a" in " ".join(_build.NVCC_FLAGS)


def test_every_declared_symbol_is_exported_and_bound():
    lib = _native.load()
    names = header_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_native.SIGNATURES) == set(names)


def test_abi_version_and_errors_without_gpu():
    lib = _native.load()
    assert lib.gs_abi_version() == _native.ABI_VERSION == 3
    # argument validation happens before any launch
    assert lib.gs_f32_to_f16(None, None, -1, 1.0, None, None) == -1
    assert b"negative" in lib.gs_last_error()
    assert lib.gs_fold_f16_tree(None, 0, 0, None, 4, None, None) == -1
    assert lib.gs_lars_pass1(None, None, 0, -1, 1, _native.StepParams(), 0, None, None, 0,
                             None, None) == -1
    # peer launches validate before touching the rank table
    assert lib.gs_rs_pass1(None, 1, 3, None, None, None, None, 0, 1, _native.StepParams(), 0, 0,
                           1, 8, None) == -1
    assert b"p must be 2, 4 or 8" in lib.gs_last_error()
    assert lib.gs_ordered_allreduce_f16(None, 1, 2, None, None, 0, 16, 0, 8, 0, None) == -1
    assert b"epoch 0" in lib.gs_last_error()
    assert lib.gs_peer_fence(None, 3, 2, None, 1, 0, None) == -1
    assert lib.gs_trust_fence(None, 1, 2, None, 0, 1, 1, _native.StepParams(), 0, None) == -1


def test_struct_layouts_match_header():
    text = (ROOT / "include" / "gradsync_b200.h").read_text()
    for dt, name, size in ((_native.SEGMENT_DTYPE, "gs_segment", 64),
                           (_native.CHUNK_DTYPE, "gs_chunk", 16),
                           (_native.COPY_DTYPE, "gs_copy", 24),
                           (_native.STEP_PARAMS_DTYPE, "gs_step_params", 56),
                           (_native.CTL_DTYPE, "gs_ctl", 48),
                           (_native.RANK_CTX_DTYPE, "gs_rank_ctx", 120)):
        assert dt.itemsize == size
        assert re.search(rf"}}\s*{name};\s*/\*\s*{size} bytes", text), name
    m = {k: int(v, 0) for k, v in re.findall(r"#define (GS_[A-Z0-9_]+) (\d+|0x[0-9a-f]+)u?", text)}
    assert m["GS_MODE_DIV1"] == _native.MODE_DIV1 and m["GS_MODE_GRADNORM"] == _native.MODE_GRADNORM
    assert m["GS_SEG_LARS_ENABLED"] == _native.SEG_LARS_ENABLED
    assert m["GS_FLAG_GRAD_NONFINITE"] == _native.FLAG_GRAD_NONFINITE


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_1807_11205_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", f.read_text(), re.M), f


def test_no_packed_fp32_contraction_in_sass():
    """ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even with
    -fmad=false; the library must not contain packed fp32 arithmetic at all,
    and the bit-exact update kernels must not contain FFMA (contracted a*b+c)
    outside the IEEE-division slow path."""
    import shutil
    import subprocess
    import pytest
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", str(_build.LIBPATH)], capture_output=True, text=True,
                          check=True).stdout
    for op in ("FFMA2", "FADD2", "FMUL2"):
        assert op not in sass
    # pass-2 specialisation for power-of-two scaling: pure FMUL/FADD
    funcs = sass.split("Function : ")
    p2 = [f for f in funcs if "lars_pass2_kernelILb1ELb1EE" in f.split("\n", 1)[0]]
    assert p2, "pow2 pass-2 kernel missing"
    assert "FFMA" not in p2[0]
