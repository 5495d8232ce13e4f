"""Peer-synchronised launches (collectives and fused collective + LARS kernels).

Every such kernel takes a device table of gs_rank_ctx (include/gradsync_b200.h):
one entry on a multi-GPU box — this GPU's rank — or p entries when the p ranks
of a job are emulated on one device (emulation.LocalWorld), in which case ONE
launch carries every rank and all their CTAs are co-resident by construction.

A pipeline describes such a launch as a :class:`PeerOp` (this rank's context
record + the arguments every rank passes identically); :func:`launch` batches
one op per rank into a single call.  The contexts are uploaded once per
distinct set and cached.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _native

__all__ = ["PeerOp", "PeerTimeoutError", "launch", "rank_ctx", "decode_status"]

#: site codes recorded in gs_ctl.status (gs_peer.cuh kSite*)
SITES = {1: "ordered all-reduce", 2: "reduce-scatter", 3: "all-gather", 4: "reduce-scatter+pass1",
         5: "peer fence", 6: "hierarchical all-reduce"}


class PeerTimeoutError(RuntimeError):
    """A peer wait exceeded its bound: some rank never reached the collective
    (it died, diverged in its call sequence, or the box is oversubscribed)."""


def decode_status(status: int) -> str:
    site = (status >> 20) & 0xFF
    return (f"rank {status & 0xFF} waited past its timeout for peer {(status >> 8) & 0xFF} "
            f"in the {SITES.get(site, f'site {site}')} kernel (barrier phase "
            f"{(status >> 16) & 0xF}); status word 0x{status:08x}")


def rank_ctx(rank: int, *, timeout_s: float = 120.0, status: int = 0, epoch_base: int = 0,
             segs: int = 0, chunks: int = 0, own_list: int = 0, own_off: int = 0, ctl: int = 0,
             seg_scale: int = 0, nonfinite: int = 0, red: int = 0, partials: int = 0,
             seg_out: int = 0, seg_ready: int = 0) -> np.ndarray:
    """One gs_rank_ctx record (addresses as ints; 0 = NULL)."""
    r = np.zeros(1, dtype=_native.RANK_CTX_DTYPE)
    r["rank"] = rank
    r["timeout_ns"] = int(timeout_s * 1e9)
    r["status"], r["epoch_base"], r["segs"], r["chunks"] = status, epoch_base, segs, chunks
    r["own_list"], r["own_off"], r["ctl"], r["seg_scale"] = own_list, own_off, ctl, seg_scale
    r["nonfinite"], r["red"] = nonfinite, red
    r["partials"], r["seg_out"], r["seg_ready"] = partials, seg_out, seg_ready
    return r


@dataclass
class PeerOp:
    """One rank's share of a peer launch: `fn(ranks, nranks, *args)`.

    `args` must be identical on every rank of a batched launch.  For
    gs_pass2_push, `count` is this rank's owned chunk count and the args
    hold None where the launch needs the maximum over ranks."""
    fn: str
    ctx: np.ndarray
    args: tuple
    count: int | None = None
    device: torch.device | None = field(default=None, compare=False)


_CACHE: dict = {}
_CACHE_MAX = 256


def _key(a):
    if isinstance(a, _native.StepParams):
        return bytes(a)
    return a


def batched_table(ctxs, device=None) -> torch.Tensor:
    """The device gs_rank_ctx table of several ranks (uploaded once per
    distinct content and cached)."""
    raw = b"".join(c.tobytes() for c in ctxs)
    tab = _CACHE.get(raw)
    if tab is None:
        if len(_CACHE) >= _CACHE_MAX:
            _CACHE.pop(next(iter(_CACHE)))
        tab = _CACHE[raw] = dev.upload(np.frombuffer(raw, dtype=np.uint8).copy(),
                                       device or torch.device("cuda", torch.cuda.current_device()))
    return tab


def launch(ops: list[PeerOp]) -> None:
    """Launch one op per rank (ranks in order) as ONE kernel call."""
    if not ops:
        return
    first = ops[0]
    key0 = tuple(_key(a) for a in first.args)
    for op in ops[1:]:
        if op.fn != first.fn or tuple(_key(a) for a in op.args) != key0:
            raise RuntimeError(f"ranks diverged at a peer launch: {first.fn} vs {op.fn} "
                               "(every rank must issue the same collective sequence)")
    tab = batched_table([op.ctx for op in ops], first.device)
    args = first.args
    if first.count is not None:
        m = max(op.count for op in ops)
        args = tuple(m if a is None else a for a in args)
    _native.call(first.fn, dev.ptr(tab), len(ops), *args)
