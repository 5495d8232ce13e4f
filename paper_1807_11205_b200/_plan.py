"""Segment / chunk tables and the three-kernel LARS launch sequence.

A *segment* is one parameter group (lars.py:92-125): pointers to its
gradient, fp32 master, fp32 velocity and binary16 working copy.  A *chunk*
is a contiguous range of one segment of at most CHUNK_ELEMS elements; one
CTA of gs_lars_pass1 / gs_lars_pass2 handles one chunk, so the chunk table
is the grid.  Chunks are laid out in the order the caller wants them
traversed (the fused pipeline uses wire order so a bucket is a contiguous
chunk range).  The fp64 partial sums of a segment are folded by
gs_lars_trust in chunk order, so results depend only on this table.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _native

#: elements per chunk: 256 threads x 8 elements x 4 unrolled rounds (the
#: pass-1 batch).  4096-element chunks with 6 CTAs/SM measured no better
#: (profiles/r02/pass1_variants.md)
CHUNK_ELEMS = 8192


def build_chunks(sizes, order=None, chunk_elems: int = CHUNK_ELEMS):
    """Chunk table over segments `sizes` traversed in `order`.

    Returns (chunks[CHUNK_DTYPE], chunk_begin[nseg], chunk_count[nseg]).
    Zero-length segments own no chunk.
    """
    sizes = [int(n) for n in sizes]
    order = list(range(len(sizes))) if order is None else list(order)
    begin = np.zeros(len(sizes), dtype=np.int32)
    count = np.zeros(len(sizes), dtype=np.int32)
    rows = []
    for s in order:
        n = sizes[s]
        begin[s] = len(rows)
        nch = (n + chunk_elems - 1) // chunk_elems
        for c in range(nch):
            st = c * chunk_elems
            rows.append((st, s, min(chunk_elems, n - st)))
        count[s] = nch
    chunks = np.zeros(len(rows), dtype=_native.CHUNK_DTYPE)
    if rows:
        arr = np.array(rows, dtype=np.int64)
        chunks["start"] = arr[:, 0]
        chunks["seg"] = arr[:, 1]
        chunks["len"] = arr[:, 2]
    return chunks, begin, count


def _pow2_rcp(d: np.float32):
    """(is_pow2, reciprocal) — x*rcp == x/d bitwise when d is a power of two
    whose reciprocal is exactly representable."""
    d = np.float32(d)
    if not np.isfinite(d) or d <= 0:
        return False, np.float32(0)
    m, _ = np.frexp(d)
    if m != 0.5:
        return False, np.float32(0)
    with np.errstate(over="ignore"):
        r = np.float32(1) / d
    ok = np.isfinite(r) and np.float32(r * d) == np.float32(1) and np.frexp(r)[0] == 0.5 \
        and r >= np.finfo(np.float32).tiny
    return bool(ok), r


def step_params(*, eta: float, epsilon: float, gamma: float, weight_decay: float,
                momentum: float, mean_divisor: float | None = None,
                unscale_divisor: float | None = None, grad_norm: bool = False) -> np.ndarray:
    """Host struct gs_step_params for one step."""
    p = np.zeros(1, dtype=_native.STEP_PARAMS_DTYPE)
    p["eta"] = float(eta)
    p["epsilon"] = float(epsilon)
    p["gamma"] = float(gamma)
    p["weight_decay"] = np.float32(weight_decay)
    p["momentum"] = np.float32(momentum)
    mode = 0
    if weight_decay != 0.0:
        mode |= _native.MODE_DECAY
    if grad_norm:
        mode |= _native.MODE_GRADNORM
    if mean_divisor is not None:
        d = np.float32(mean_divisor)
        pw, r = _pow2_rcp(d)
        p["div1"], p["rcp1"] = d, r
        mode |= _native.MODE_DIV1 | (_native.MODE_DIV1_POW2 if pw else 0)
    if unscale_divisor is not None:
        d = np.float32(unscale_divisor)
        pw, r = _pow2_rcp(d)
        p["div2"], p["rcp2"] = d, r
        mode |= _native.MODE_DIV2 | (_native.MODE_DIV2_POW2 if pw else 0)
    p["mode"] = mode
    return p


def launch_hint(p: np.ndarray, g_is_f16: bool) -> int:
    """GS_HINT_* bits for a step-params struct, filling in `mul`.

    POW2: the mean and unscale divisions are exact power-of-two scalings that
    compose into one multiplication: for fp16 input every widened value is
    0 or >= 2^-24 in magnitude, so x * rcp1 is exact and x*rcp1*rcp2 rounds
    once either way.  fp32 input qualifies only without divisors.
    RAWFLAG: fp16 input and mul <= 1, so no finite value can overflow and the
    finite tests reduce to the binary16 exponent field.
    """
    mode = int(p["mode"][0])
    div1, div2 = mode & _native.MODE_DIV1, mode & _native.MODE_DIV2
    ok = g_is_f16 or not (div1 or div2)
    if div1 and not mode & _native.MODE_DIV1_POW2:
        ok = False
    if div2 and not mode & _native.MODE_DIV2_POW2:
        ok = False
    hint = _native.HINT_GRADNORM if mode & _native.MODE_GRADNORM else 0
    if ok:
        mul = (float(p["rcp1"][0]) if div1 else 1.0) * (float(p["rcp2"][0]) if div2 else 1.0)
        if 2.0 ** -100 <= mul <= 2.0 ** 100:
            p["mul"] = np.float32(mul)
            hint |= _native.HINT_POW2
            if g_is_f16 and mul <= 1.0:
                hint |= _native.HINT_RAWFLAG
    return hint


@dataclass
class SegmentSpec:
    g: int
    w: int
    v: int
    w16: int
    n: int
    flags: int


class LarsPlan:
    """Device tables + scratch for running pass1 -> trust -> pass2 over a
    fixed set of segments.

    The step scalars are passed by value to every kernel (no per-step
    host->device copy).  The flag words live in a gs_ctl block, double-
    buffered by step parity: step k (``self.seq``) uses index k & 1 and its
    trust kernel clears index (k + 1) & 1 for the next step; ``end_step()``
    advances k.  ``ctl`` may be supplied (the sharded update keeps it in the
    symmetric window so peers can OR their flags into it)."""

    def __init__(self, specs: list[SegmentSpec], device: torch.device, order=None,
                 chunk_elems: int = CHUNK_ELEMS, partials: torch.Tensor | None = None,
                 ctl: torch.Tensor | None = None):
        self.device = device
        self.nseg = len(specs)
        chunks, begin, count = build_chunks([s.n for s in specs], order, chunk_elems)
        segs = np.zeros(self.nseg, dtype=_native.SEGMENT_DTYPE)
        for i, s in enumerate(specs):
            segs[i]["g"], segs[i]["w"], segs[i]["v"], segs[i]["w16"] = s.g, s.w, s.v, s.w16
            segs[i]["n"] = s.n
            segs[i]["flags"] = s.flags
        segs["chunk_begin"] = begin
        segs["chunk_count"] = count
        self.host_segs, self.host_chunks = segs, chunks
        self.nchunk = len(chunks)
        self.d_segs = dev.upload(segs, device)
        self.base_segs = self.d_segs
        self._alt: dict = {}
        self.d_chunks = dev.upload(chunks, device)
        self.partials = partials if partials is not None else \
            torch.zeros(max(1, 3 * self.nchunk), dtype=torch.float64, device=device)
        self.seg_scale = torch.zeros(max(1, self.nseg), dtype=torch.float32, device=device)
        self.seg_out = torch.zeros(max(1, 4 * self.nseg), dtype=torch.float64, device=device)
        csz = _native.CTL_DTYPE.itemsize
        self.ctl = ctl if ctl is not None else torch.zeros(csz, dtype=torch.uint8, device=device)
        assert self.ctl.numel() * self.ctl.element_size() >= csz
        self._ctl_host = torch.zeros(csz, dtype=torch.uint8).pin_memory()
        #: step sequence number (parity = seq & 1 selects the flag word)
        self.seq = 0
        #: per-chunk sum w^2 carried from pass 2 to the next step's pass 1
        #: (enable_w2_cache); valid only while nothing else writes the masters
        self.wsq = None
        self.wsq_valid = False
        self.hint = 0
        self.sp = _native.StepParams()
        self.params_np = np.zeros(1, dtype=_native.STEP_PARAMS_DTYPE)

    def enable_w2_cache(self) -> None:
        """Let pass 2 leave the updated masters' per-chunk sum w^2 for the
        next step's pass 1 (for owners of the master arena: the pipeline)."""
        if self.wsq is None:
            self.wsq = torch.full((max(1, self.nchunk),), float("nan"), dtype=torch.float64,
                                  device=self.device)

    def invalidate_w2_cache(self) -> None:
        """The masters changed outside pass 2: the next pass 1 re-derives w^2."""
        self.wsq_valid = False

    @property
    def parity(self) -> int:
        return self.seq & 1

    def end_step(self) -> None:
        self.seq += 1

    def alt_segments(self, g_ptrs) -> torch.Tensor:
        """A segment table identical to the base one except for the gradient
        pointers, uploaded once per pointer set (bounded cache)."""
        key = tuple(g_ptrs)
        tab = self._alt.get(key)
        if tab is None:
            segs = self.host_segs.copy()
            segs["g"] = np.asarray(g_ptrs, dtype=np.uint64)
            if len(self._alt) >= 16:
                self._alt.pop(next(iter(self._alt)))
            tab = self._alt[key] = dev.upload(segs, self.device)
        return tab

    def use_segments(self, table: torch.Tensor | None) -> None:
        """Select the segment table the next launches run over (None = base)."""
        self.d_segs = self.base_segs if table is None else table

    # -- individual launches (all async on `stream`) --------------------
    def set_params(self, params: np.ndarray, g_is_f16: bool = False) -> int:
        """The step scalars of the next launches (host only: they travel by
        value) and the launch hint derived from them."""
        self.hint = launch_hint(params, g_is_f16)
        self.params_np = params.copy()
        self.sp = _native.StepParams.of(params)
        return self.hint

    def reset_flags(self, stream_h: int) -> None:
        """Zero both flag words and counters (only needed after a step that
        ran pass 1 without trust, e.g. lars_step's gate-only probe)."""
        _native.call("gs_fill_zero", dev.ptr(self.ctl), 16, stream_h)

    def pass1(self, stream_h: int, g_is_f16: bool, chunk0: int = 0, nchunk: int | None = None):
        n = self.nchunk - chunk0 if nchunk is None else nchunk
        _native.call("gs_lars_pass1", dev.ptr(self.d_segs), dev.ptr(self.d_chunks), chunk0, n,
                     1 if g_is_f16 else 0, self.sp, self.hint, dev.ptr(self.partials),
                     dev.ptr(self.ctl), self.parity,
                     dev.ptr(self.wsq) if self.wsq_valid else None, stream_h)

    def trust(self, stream_h: int, peer_ctl: torch.Tensor | None = None, npeers: int = 0):
        _native.call("gs_lars_trust", dev.ptr(self.d_segs), self.nseg, self.nchunk,
                     dev.ptr(self.partials),
                     self.sp, dev.ptr(self.seg_scale), dev.ptr(self.seg_out), dev.ptr(self.ctl),
                     self.parity, dev.ptr(peer_ctl) if peer_ctl is not None else None, npeers,
                     stream_h)

    def pass2(self, stream_h: int, g_is_f16: bool, flag_mask: int, chunk0: int = 0,
              nchunk: int | None = None):
        n = self.nchunk - chunk0 if nchunk is None else nchunk
        _native.call("gs_lars_pass2", dev.ptr(self.d_segs), dev.ptr(self.d_chunks), chunk0, n,
                     1 if g_is_f16 else 0, self.sp, self.hint, dev.ptr(self.seg_scale),
                     dev.ptr(self.ctl), self.parity, flag_mask,
                     dev.ptr(self.wsq) if self.wsq is not None else None, stream_h)

    def finish(self, stream_h: int, g_is_f16: bool, flag_mask: int) -> None:
        """trust + pass 2 (pass 2 is a programmatic dependent of trust)."""
        self.trust(stream_h)
        self.pass2(stream_h, g_is_f16, flag_mask)

    def run(self, stream_h: int, g_is_f16: bool, flag_mask: int) -> None:
        """One whole step: pass 1 -> trust -> pass 2, then advance the parity."""
        self.pass1(stream_h, g_is_f16)
        self.finish(stream_h, g_is_f16, flag_mask)
        self.end_step()

    def read_ctl(self, stream=None) -> np.void:
        """Copy the control block to the host (syncs `stream`) and return it
        as a CTL_DTYPE record: flags[parity], status, grad_norm."""
        s = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            self._ctl_host.copy_(self.ctl.view(torch.uint8)[: self._ctl_host.numel()],
                                 non_blocking=True)
        s.synchronize()
        return self._ctl_host.numpy().view(_native.CTL_DTYPE)[0]

    def last_flags(self, rec) -> int:
        """Flags of the last completed step (end_step() already advanced)."""
        return int(rec["flags"][(self.seq - 1) & 1])
