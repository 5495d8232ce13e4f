"""Frozen parameter-shape lists and the seeded synthetic-input generator.

shapes.json was frozen from torchvision's model definitions (no weights):
  resnet50            161 tensors, 25 557 032 params (54 weight, 1 bias, 53+53 BN)
  alexnet              16 tensors, 61 100 840 params (8 weight, 8 bias)
  shufflenet_v2_x0_5  170 tensors,  1 366 792 params (57 weight, 1 bias, 56+56 BN)
Kind map: BN .weight -> bn_gamma, BN .bias -> bn_beta, other
dim>1 -> weight, other 1-D -> bias.

Synthetic inputs: every tensor draws from
np.random.default_rng([seed, stream, tensor_index]) so any subset of ranks or
tensors can be regenerated independently; master weights ~ N(0, sqrt(2/fan_in))
for weights, gamma = 1, beta = 0, biases ~ N(0, 0.01); per-rank true
gradients ~ N(0, 1e-3) in fp32; the wire gradient of rank r is
binary16(RNE(g * loss_scale)), as a mixed-precision backward would produce.
"""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from .pipeline import ParamSpec

_PATH = Path(__file__).with_name("shapes.json")
MODELS = ("resnet50", "alexnet", "shufflenet_v2_x0_5")
WEIGHT_STREAM = 1 << 20


@lru_cache(maxsize=None)
def _table() -> dict:
    return json.loads(_PATH.read_text())


def load_shapes(model: str) -> list[ParamSpec]:
    if model not in _table():
        raise KeyError(f"unknown model {model!r}; have {sorted(_table())}")
    return [ParamSpec(name, tuple(shape), kind) for name, shape, kind in _table()[model]]


def total_params(specs) -> int:
    return int(sum(s.numel for s in specs))


def synth_master(specs, seed: int = 0) -> np.ndarray:
    """Flat fp32 master weights in registration order."""
    out = np.empty(total_params(specs), dtype=np.float32)
    o = 0
    for i, s in enumerate(specs):
        n = s.numel
        rng = np.random.default_rng([seed, WEIGHT_STREAM, i])
        if s.kind == "weight":
            fan_in = int(np.prod(s.shape[1:])) if len(s.shape) > 1 else 1
            out[o:o + n] = rng.standard_normal(n, dtype=np.float32) * np.float32(np.sqrt(2.0 / fan_in))
        elif s.kind == "bn_gamma":
            out[o:o + n] = 1.0
        elif s.kind == "bn_beta":
            out[o:o + n] = 0.0
        else:
            out[o:o + n] = rng.standard_normal(n, dtype=np.float32) * np.float32(0.01)
        o += n
    return out


def synth_grads_f32(specs, rank: int, seed: int = 0, sigma: float = 1e-3) -> np.ndarray:
    """Flat fp32 'true' gradients of one rank in registration order."""
    out = np.empty(total_params(specs), dtype=np.float32)
    o = 0
    for i, s in enumerate(specs):
        n = s.numel
        rng = np.random.default_rng([seed, rank, i])
        out[o:o + n] = rng.standard_normal(n, dtype=np.float32) * np.float32(sigma)
        o += n
    return out


def synth_wire_grads(specs, rank: int, seed: int = 0, loss_scale: float = 1024.0,
                     sigma: float = 1e-3) -> np.ndarray:
    """Flat uint16 binary16 wire gradients of one rank: RNE(g * scale).

    numpy's float32->float16 cast is IEEE RNE; no NaN can occur here, so it
    equals the reference narrowing (halfprec.py:40-85) bit for bit.
    """
    g = synth_grads_f32(specs, rank, seed, sigma) * np.float32(loss_scale)
    with np.errstate(over="ignore"):
        return g.astype(np.float16).view(np.uint16)
