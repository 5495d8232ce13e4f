"""ctypes binding of libgradsync_b200.so (C ABI in include/gradsync_b200.h).

There is no CPU fallback: any device arithmetic goes through this library,
and ``lib()`` raises if the shared object is missing or cannot be loaded.
Host-only bookkeeping (fusion planning, schedules, validation) never needs it.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_double, c_float, c_int, c_int64, c_uint32, c_void_p

import numpy as np

from . import _build

GS_OK = 0

SEG_DECAY_EXEMPT = 1
SEG_LARS_ENABLED = 2

MODE_DIV1 = 1
MODE_DIV1_POW2 = 2
MODE_DIV2 = 4
MODE_DIV2_POW2 = 8
MODE_DECAY = 16
MODE_GRADNORM = 32

FLAG_SCALED_NONFINITE = 1
FLAG_GRAD_NONFINITE = 2

HINT_POW2 = 1
HINT_RAWFLAG = 2
HINT_GRADNORM = 4

# numpy mirrors of the device structs (layout asserted against the header)
SEGMENT_DTYPE = np.dtype([
    ("g", "<u8"), ("w", "<u8"), ("v", "<u8"), ("w16", "<u8"),
    ("n", "<i8"), ("chunk_begin", "<i4"), ("chunk_count", "<i4"),
    ("flags", "<u4"), ("reserved", "<u4"), ("reserved2", "<u8"),
])
CHUNK_DTYPE = np.dtype([("start", "<i8"), ("seg", "<i4"), ("len", "<i4")])
COPY_DTYPE = np.dtype([("src", "<u8"), ("dst", "<u8"), ("nbytes", "<i8")])
STEP_PARAMS_DTYPE = np.dtype([
    ("eta", "<f8"), ("epsilon", "<f8"), ("gamma", "<f8"),
    ("weight_decay", "<f4"), ("momentum", "<f4"),
    ("div1", "<f4"), ("rcp1", "<f4"), ("div2", "<f4"), ("rcp2", "<f4"),
    ("mode", "<u4"), ("mul", "<f4"),
])
CTL_DTYPE = np.dtype([
    ("flags", "<u4", (2,)), ("counter", "<u4", (2,)), ("status", "<u4"), ("reserved", "<u4", (3,)),
    ("grad_norm", "<f8"), ("reserved2", "<f8"),
])
RANK_CTX_DTYPE = np.dtype([
    ("rank", "<i4"), ("reserved", "<i4"), ("timeout_ns", "<u8"), ("status", "<u8"),
    ("epoch_base", "<u8"), ("segs", "<u8"), ("chunks", "<u8"), ("own_list", "<u8"),
    ("own_off", "<u8"), ("ctl", "<u8"), ("seg_scale", "<u8"), ("nonfinite", "<u8"),
    ("red", "<u8"), ("partials", "<u8"), ("seg_out", "<u8"), ("seg_ready", "<u8"),
])
STEP_RANK_DTYPE = np.dtype([
    ("pack", "<u8"), ("npack", "<i4"), ("nseg", "<i4"), ("segs", "<u8"), ("chunks", "<u8"),
    ("nchunk", "<i4"), ("reserved", "<i4"), ("partials", "<u8"), ("seg_scale", "<u8"),
    ("seg_out", "<u8"), ("ctl", "<u8"), ("wsq_in", "<u8"), ("wsq_out", "<u8"),
    ("epoch_base", "<u8"),
])
assert STEP_RANK_DTYPE.itemsize == 96
assert SEGMENT_DTYPE.itemsize == 64
assert CTL_DTYPE.itemsize == 48
assert RANK_CTX_DTYPE.itemsize == 120
assert CHUNK_DTYPE.itemsize == 16
assert COPY_DTYPE.itemsize == 24
assert STEP_PARAMS_DTYPE.itemsize == 56


class StepParams(ctypes.Structure):
    """gs_step_params, passed BY VALUE to the LARS / fused kernels."""
    _fields_ = [("eta", c_double), ("epsilon", c_double), ("gamma", c_double),
                ("weight_decay", c_float), ("momentum", c_float),
                ("div1", c_float), ("rcp1", c_float), ("div2", c_float), ("rcp2", c_float),
                ("mode", c_uint32), ("mul", c_float)]

    @classmethod
    def of(cls, p: np.ndarray) -> "StepParams":
        return cls.from_buffer_copy(np.ascontiguousarray(p).view(np.uint8).tobytes())


assert ctypes.sizeof(StepParams) == STEP_PARAMS_DTYPE.itemsize

#: every symbol include/gradsync_b200.h declares, with its ctypes signature
SIGNATURES = {
    "gs_abi_version": (c_int, []),
    "gs_kernel_launches": (c_int64, []),
    "gs_last_error": (ctypes.c_char_p, []),
    "gs_device_sm_count": (c_int, [c_int]),
    "gs_f32_to_f16": (c_int, [c_void_p, c_void_p, c_int64, c_float, c_void_p, c_void_p]),
    "gs_f16_to_f32": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "gs_quantize_f32": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "gs_unscale_f32": (c_int, [c_void_p, c_void_p, c_int64, c_float, c_void_p]),
    "gs_nonfinite": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int, c_void_p, c_uint32,
                             c_void_p]),
    "gs_batched_copy": (c_int, [c_void_p, c_int, c_void_p]),
    "gs_fold_f32": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_int, c_void_p]),
    "gs_fold_f16_tree": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p,
                                 c_void_p]),
    "gs_lars_pass1": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, StepParams, c_uint32,
                              c_void_p, c_void_p, c_uint32, c_void_p, c_void_p]),
    "gs_lars_trust": (c_int, [c_void_p, c_int, c_int, c_void_p, StepParams, c_void_p, c_void_p,
                              c_void_p, c_uint32, c_void_p, c_int, c_void_p]),
    "gs_lars_pass2": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, StepParams, c_uint32,
                              c_void_p, c_void_p, c_uint32, c_uint32, c_void_p, c_void_p]),
    "gs_fill_zero": (c_int, [c_void_p, c_int64, c_void_p]),
    "gs_ordered_allreduce_f16": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int64,
                                         c_int64, c_uint32, c_int, c_int, c_void_p]),
    "gs_ordered_allreduce_f32": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int64,
                                         c_int64, c_uint32, c_int, c_int, c_void_p]),
    "gs_oneshot_allreduce_f16": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                         c_int64, c_int64, c_int64, c_uint32, c_int, c_uint32,
                                         c_void_p]),
    "gs_ll_allreduce_f16": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int64, c_int64,
                                    c_int64, c_uint32, c_int, c_uint32, c_void_p]),
    "gs_hier_allreduce_f16": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int64,
                                      c_int64, c_uint32, c_int, c_int, c_void_p]),
    "gs_ordered_reduce_scatter_f16": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p,
                                              c_void_p, c_uint32, c_int, c_void_p]),
    "gs_ordered_allgather": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                     c_uint32, c_int, c_void_p]),
    "gs_counter_add": (c_int, [c_void_p, c_uint32, c_void_p]),
    "gs_rs_pass1": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                            c_int, c_int, StepParams, c_uint32, c_uint32, c_uint32, c_int,
                            c_void_p]),
    "gs_pass2_push": (c_int, [c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_int, StepParams,
                              c_uint32, c_uint32, c_uint32, c_void_p]),
    "gs_zero_update": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_uint32, c_int, c_int,
                               c_int, c_int, c_int, StepParams, c_uint32, c_uint32, c_uint32,
                               c_void_p]),
    "gs_trust_fence": (c_int, [c_void_p, c_int, c_int, c_void_p, c_uint32, c_int, c_int,
                               StepParams, c_uint32, c_void_p]),
    "gs_peer_fence": (c_int, [c_void_p, c_int, c_int, c_void_p, c_uint32, c_uint32, c_void_p]),
    "gs_step_replicated": (c_int, [c_void_p, c_int, StepParams, c_uint32, c_uint32, c_uint32,
                                   c_void_p]),
    "gs_step_zero": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                             c_void_p, c_void_p, c_int, c_int, StepParams, c_uint32, c_uint32,
                             c_uint32, c_int, c_void_p]),
}

ABI_VERSION = 3

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A libgradsync_b200 call returned a non-zero status."""


def library_path() -> str:
    return os.environ.get("GRADSYNC_B200_LIB", str(_build.LIBPATH))


def load(path: str | None = None) -> ctypes.CDLL:
    """Load the shared library and bind every declared symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or library_path()
        if not os.path.exists(p):
            raise NativeError(
                f"libgradsync_b200 not built ({p} missing); run "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
        cdll = ctypes.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(cdll, name)  # AttributeError = missing export
            fn.restype = res
            fn.argtypes = args
        if cdll.gs_abi_version() != ABI_VERSION:
            raise NativeError(f"ABI mismatch: library {cdll.gs_abi_version()} != {ABI_VERSION}")
        if path is None:
            _lib = cdll
        return cdll


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load()


def check(status: int, what: str) -> None:
    if status != GS_OK:
        msg = lib().gs_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({status}): {msg}")


#: entry points that launch a kernel (everything but the queries)
_LAUNCHING = {n for n in SIGNATURES if n not in ("gs_abi_version", "gs_last_error",
                                                 "gs_device_sm_count", "gs_kernel_launches")}
#: running count of kernel-launching calls (bench.py's gpu_launches evidence)
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    check(getattr(lib(), name)(*args), name)
    if name in _LAUNCHING:
        launch_count += 1


def kernel_launches() -> int:
    """Kernels the library has launched in this process (counted in C at
    every launch site, so one gs_step_* call counts each of its kernels)."""
    return int(lib().gs_kernel_launches())


def stream_handle(stream=None) -> int:
    """cudaStream_t of `stream` (default: torch's current stream)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
