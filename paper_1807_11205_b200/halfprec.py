"""IEEE binary16 conversions and loss scaling (drop-in for gradsync.halfprec).

Reference: pkg/src/gradsync/halfprec.py.  FP16 data is carried as uint16 bit
patterns exactly as in the reference (halfprec.py:3-7); the conversions run
as libgradsync_b200 kernels (gs_f32_to_f16 / gs_f16_to_f32 / gs_quantize_f32 /
gs_unscale_f32 / gs_nonfinite).  Narrowing is IEEE round-to-nearest-even with
overflow to +-Inf, magnitudes below 2**-25 to signed zero and every NaN to
0x7E00 — the reference's `_narrow_bits` (halfprec.py:40-85) equals hardware
RNE on every non-NaN float32 pattern, so the kernel is bit-exact.

Inputs may be numpy arrays/scalars (the result is returned as numpy, like the
reference) or CUDA tensors (the result stays on the device).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _native

__all__ = [
    "SMALLEST_SUBNORMAL",
    "FLUSH_BOUND",
    "MAX_FINITE",
    "CANONICAL_NAN",
    "f32_to_f16",
    "f16_to_f32",
    "quantize_tensor",
    "describe_half",
    "LossScale",
    "apply_loss_scale",
    "unscale_gradients",
]

#: Smallest positive binary16 value, 2**-24 (halfprec.py:30-31).
SMALLEST_SUBNORMAL = 2.0 ** -24
#: Magnitudes strictly below this become signed zero when narrowing.
FLUSH_BOUND = 2.0 ** -25
#: Largest finite binary16 value.
MAX_FINITE = 65504.0
#: Every NaN narrows to this single quiet pattern (halfprec.py:36-37).
CANONICAL_NAN = np.uint16(0x7E00)


def _run_unary(values, in_dtype, out_dtype, launch):
    """Shared numpy/tensor plumbing for the elementwise conversion kernels."""
    if dev.is_tensor(values):
        x = values
        if x.dtype != in_dtype:
            x = x.to(in_dtype)
        x = dev.to_cuda(x)
        out = torch.empty(x.shape, dtype=out_dtype, device=x.device)
        launch(x, out)
        return out
    a = np.asarray(values, dtype=dev._TORCH_TO_NP[in_dtype])
    x = dev.to_cuda(a.reshape(-1))
    out = torch.empty(x.shape, dtype=out_dtype, device=x.device)
    launch(x, out)
    res = dev.to_host(out).reshape(a.shape)
    return res[()] if a.ndim == 0 else res


def f32_to_f16(values, *, scale: float = 1.0, nonfinite: torch.Tensor | None = None):
    """Narrow float32 values to binary16 bit patterns (halfprec.py:108-121).

    ``scale`` (keyword-only extension) multiplies in float32 before the
    narrowing, fusing the reference's ``f32_to_f16(g * np.float32(s))``
    (test_halfprec.py:202-210).  ``nonfinite`` (a CUDA uint32 tensor) gets 1
    OR-ed in when any output is Inf/NaN.
    """
    s = float(np.float32(scale))

    def launch(x, out):
        _native.call("gs_f32_to_f16", dev.ptr(x), dev.ptr(out), x.numel(), s,
                     dev.ptr(nonfinite) if nonfinite is not None else None, dev.stream_of())

    return _run_unary(values, torch.float32, torch.uint16, launch)


def _as_bits(bits):
    if dev.is_tensor(bits):
        if bits.dtype == torch.uint16:
            return bits
        if bits.dtype == torch.float16:
            return bits.view(torch.uint16)
        if bits.dtype.is_floating_point or bits.dtype == torch.bool:
            raise TypeError(f"expected uint16 bit patterns, got {bits.dtype}")
        return bits.to(torch.int32).bitwise_and(0xFFFF).to(torch.uint16)
    a = np.asarray(bits)
    if a.dtype != np.uint16:
        if not np.issubdtype(a.dtype, np.integer):
            raise TypeError(f"expected uint16 bit patterns, got {a.dtype}")
        a = a.astype(np.uint16)
    return a


def f16_to_f32(bits):
    """Widen binary16 bit patterns to float32 values, exactly (halfprec.py:124-132)."""
    b = _as_bits(bits)

    def launch(h, out):
        _native.call("gs_f16_to_f32", dev.ptr(h), dev.ptr(out), h.numel(), dev.stream_of())

    return _run_unary(b, torch.uint16, torch.float32, launch)


def quantize_tensor(values):
    """Round-trip float32 data through binary16 (halfprec.py:135-137)."""

    def launch(x, out):
        _native.call("gs_quantize_f32", dev.ptr(x), dev.ptr(out), x.numel(), dev.stream_of())

    return _run_unary(values, torch.float32, torch.float32, launch)


_CATEGORIES = ("zero", "subnormal", "normal", "inf", "nan")


def describe_half(bits: int) -> dict:
    """Decompose one binary16 pattern into its fields (halfprec.py:143-167).

    Pure host bookkeeping; the value is the exact rational the pattern
    encodes, computed with integer arithmetic.
    """
    b = int(bits)
    if not 0 <= b <= 0xFFFF:
        raise ValueError(f"not a 16-bit pattern: {bits!r}")
    sign = (b >> 15) & 1
    exp = (b >> 10) & 0x1F
    man = b & 0x3FF
    if exp == 31:
        category = "nan" if man else "inf"
        value = float("nan") if man else (-1.0) ** sign * float("inf")
    else:
        category = ("subnormal" if man else "zero") if exp == 0 else "normal"
        mag = (man * 2.0 ** -24) if exp == 0 else ((1024 + man) * 2.0 ** (exp - 25))
        value = -mag if sign else mag
    return {
        "bits": f"0x{b:04X}",
        "sign": sign,
        "exponent_field": exp,
        "mantissa_field": man,
        "category": category,
        "value": float(np.float32(value)),
    }


def any_nonfinite(arrays, *, is_f16: bool | None = None) -> bool:
    """True when any element of any array is Inf/NaN (one kernel + one sync)."""
    tensors = [dev.to_cuda(a) for a in arrays]
    if not tensors:
        return False
    device = tensors[0].device
    if is_f16 is None:
        is_f16 = tensors[0].dtype in (torch.uint16, torch.float16)
    want = (torch.uint16, torch.float16) if is_f16 else (torch.float32,)
    tensors = [t if t.dtype in want else t.to(torch.float32) for t in tensors]
    tensors = [t.to(device).reshape(-1) for t in tensors]
    ptrs = np.array([t.data_ptr() for t in tensors], dtype=np.uint64)
    lens = np.array([t.numel() for t in tensors], dtype=np.int64)
    tab_p = dev.upload(ptrs, device)
    tab_l = dev.upload(lens, device)
    flag = torch.zeros(1, dtype=torch.int32, device=device)
    _native.call("gs_nonfinite", dev.ptr(tab_p), dev.ptr(tab_l), len(tensors), int(lens.max()),
                 1 if is_f16 else 0, dev.ptr(flag), 1, dev.stream_of())
    return bool(flag.item())


@dataclass
class LossScale:
    """Loss-scaling state for the mixed-precision pipeline (halfprec.py:170-221).

    Host state exactly as the reference; the finite test runs on the device.
    Under the dynamic policy a non-finite gradient skips the step and halves
    the scale; ``growth_interval`` consecutive clean steps double it.
    """

    scale: float = 2.0 ** 10
    policy: str = "dynamic"
    growth_factor: float = 2.0
    backoff_factor: float = 0.5
    growth_interval: int = 200
    clean_steps: int = 0

    def __post_init__(self):
        if self.scale <= 0:
            raise ValueError(f"loss scale must stay positive, got {self.scale}")
        if self.policy not in ("fixed", "dynamic"):
            raise ValueError(f"unknown loss-scale policy {self.policy!r}")
        if self.growth_factor <= 1 or not 0 < self.backoff_factor < 1:
            raise ValueError("growth factor must exceed 1 and backoff lie in (0, 1)")
        if self.growth_interval < 1:
            raise ValueError("growth interval must be at least 1")

    def update(self, grads) -> bool:
        """Inspect this step's (still scaled) gradients and adjust the scale."""
        single = isinstance(grads, np.ndarray) or dev.is_tensor(grads)
        arrays = [grads] if single else list(grads)
        return self.update_from_flag(any_nonfinite(arrays, is_f16=False) if arrays else False)

    def update_from_flag(self, nonfinite: bool) -> bool:
        """State transition of ``update`` given the device's non-finite flag
        (halfprec.py:211-221); used by the fused pipeline, whose pass-1 kernel
        computes the flag on the fly."""
        finite = not nonfinite
        if self.policy == "fixed":
            return finite
        if not finite:
            self.scale *= self.backoff_factor
            self.clean_steps = 0
            return False
        self.clean_steps += 1
        if self.clean_steps >= self.growth_interval:
            self.scale *= self.growth_factor
            self.clean_steps = 0
        return True


def apply_loss_scale(loss: float, s) -> float:
    """Multiply the loss by the current scale (halfprec.py:224-227)."""
    scale = s.scale if isinstance(s, LossScale) else float(s)
    return loss * scale


def unscale_gradients(g, s):
    """float32(g) / float32(scale), IEEE division, new array (halfprec.py:230-234)."""
    scale = s.scale if isinstance(s, LossScale) else float(s)
    sc = float(np.float32(scale))

    def launch(x, out):
        _native.call("gs_unscale_f32", dev.ptr(x), dev.ptr(out), x.numel(), sc, dev.stream_of())

    return _run_unary(g, torch.float32, torch.float32, launch)
