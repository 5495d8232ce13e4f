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

#: elements per chunk: 256 threads x 8 elements x 4 unrolled rounds
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
    gcopy: int = 0


class LarsPlan:
    """Device tables + scratch for running pass1 -> trust -> pass2 over a
    fixed set of segments."""

    def __init__(self, specs: list[SegmentSpec], device: torch.device, order=None,
                 chunk_elems: int = CHUNK_ELEMS, partials: torch.Tensor | None = None,
                 flagbuf: torch.Tensor | None = None):
        self.device = device
        self.nseg = len(specs)
        chunks, begin, count = build_chunks([s.n for s in specs], order, chunk_elems)
        segs = np.zeros(self.nseg, dtype=_native.SEGMENT_DTYPE)
        for i, s in enumerate(specs):
            segs[i]["g"], segs[i]["w"], segs[i]["v"], segs[i]["w16"] = s.g, s.w, s.v, s.w16
            segs[i]["n"] = s.n
            segs[i]["flags"] = s.flags
            segs[i]["gcopy"] = s.gcopy
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
        self.grad_norm = torch.zeros(1, dtype=torch.float64, device=device)
        # one int32 block, reset by one kernel per step: [0] = non-finite
        # flags, [4 : 4 + nseg + 1] = per-segment / global arrival counters
        # of the fused pass1 + trust kernel
        # the step scalars and (when the plan owns it) the flag block share one
        # device allocation, [params | pad | flags], uploaded by ONE copy per
        # step whose zero tail resets the flags — no separate reset launch
        psz = _native.STEP_PARAMS_DTYPE.itemsize
        pad = (psz + 15) // 16 * 16
        nflag = 4 + self.nseg + 1
        own_flags = flagbuf is None
        ctl_bytes = pad + 4 * nflag if own_flags else psz
        self._ctl = torch.zeros(ctl_bytes, dtype=torch.uint8, device=device)
        self._pinned_ctl = torch.zeros(ctl_bytes, dtype=torch.uint8).pin_memory()
        self.params = self._ctl[:psz]
        self._pinned_params = self._pinned_ctl[:psz]
        self.flagbuf = self._ctl[pad:].view(torch.int32) if own_flags else flagbuf
        self._flags_in_ctl = own_flags
        self._ctl_fresh = False
        self.flags = self.flagbuf[0:1]
        self.counters = self.flagbuf[4:]
        self.nseg_active = int((count > 0).sum())
        self.hint = 0
        # pass 1 runs the register-staged kernel by default: on B200 it beats
        # the TMA-pipelined persistent kernel (43 vs 47 us on ResNet-50,
        # tools/pass1_variants.py); clear HINT_NO_BULK to select the latter
        self.extra_hint = _native.HINT_NO_BULK
        # the trust ratio as a separate single-CTA kernel: fusing it into
        # pass 1 through per-chunk arrival counters costs a release atomic
        # per chunk on the critical path (61 vs 43 us); see DESIGN.md §4
        self.fuse_trust = False
        # the trust ratio folded into pass 2 (each CTA re-derives its
        # segment's scale) measured no faster than the separate trust kernel
        # chained to pass 2 by programmatic dependent launch; DESIGN.md §4
        self.trust_in_pass2 = False

    def alt_segments(self, g_ptrs, gcopy_ptrs=None) -> torch.Tensor:
        """A segment table identical to the base one except for the gradient
        (and gcopy) pointers, uploaded once per pointer set and cached."""
        key = (tuple(g_ptrs), tuple(gcopy_ptrs) if gcopy_ptrs is not None else None)
        tab = self._alt.get(key)
        if tab is None:
            segs = self.host_segs.copy()
            segs["g"] = np.asarray(g_ptrs, dtype=np.uint64)
            if gcopy_ptrs is not None:
                segs["gcopy"] = np.asarray(gcopy_ptrs, dtype=np.uint64)
            if len(self._alt) > 8:
                self._alt.clear()
            tab = self._alt[key] = dev.upload(segs, self.device)
        return tab

    def use_segments(self, table: torch.Tensor | None) -> None:
        """Select the segment table the next launches run over (None = base)."""
        self.d_segs = self.base_segs if table is None else table

    # -- individual launches (all async on `stream`) --------------------
    def set_params(self, params: np.ndarray, stream=None, g_is_f16: bool = False) -> None:
        """Stage the step scalars into the device struct and derive the launch
        hint.  The pinned staging buffer is reused, so the caller must not call
        this again before the previous copy executed (lars_step and the
        pipeline both sync on the step's flags every step)."""
        self.stage_params(params, g_is_f16)
        self.upload_params(stream)

    def stage_params(self, params: np.ndarray, g_is_f16: bool = False) -> int:
        """Host half of set_params: hint + pinned staging (no CUDA call)."""
        self.hint = launch_hint(params, g_is_f16) | self.extra_hint
        self._pinned_params.numpy()[:] = params.view(np.uint8).reshape(-1)
        return self.hint

    def upload_params(self, stream=None) -> None:
        """Device half of set_params: one async copy of the step scalars and,
        when the plan owns the flag block, of its zeros (the flag reset)."""
        s = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            self._ctl.copy_(self._pinned_ctl, non_blocking=True)
        self._ctl_fresh = self._flags_in_ctl

    def reset_flags(self, stream_h: int) -> None:
        """Zero the flag block, unless the step's parameter upload just did."""
        if self._ctl_fresh:
            self._ctl_fresh = False
            return
        _native.call("gs_fill_zero", dev.ptr(self.flagbuf), 4 * self.flagbuf.numel(), stream_h)

    @property
    def fused(self) -> bool:
        """pass1 computes the trust ratios itself (no separate trust launch)."""
        return self.fuse_trust and self.nseg_active > 0

    def pass1(self, stream_h: int, g_is_f16: bool, chunk0: int = 0, nchunk: int | None = None,
              fuse: bool = True):
        n = self.nchunk - chunk0 if nchunk is None else nchunk
        if fuse and self.fused:
            _native.call("gs_lars_pass1_trust", dev.ptr(self.d_segs), self.nseg, self.nseg_active,
                         dev.ptr(self.d_chunks), chunk0, n, 1 if g_is_f16 else 0,
                         dev.ptr(self.params), self.hint, dev.ptr(self.partials), dev.ptr(self.flags),
                         dev.ptr(self.counters), dev.ptr(self.seg_scale), dev.ptr(self.seg_out),
                         dev.ptr(self.grad_norm), stream_h)
        else:
            _native.call("gs_lars_pass1", dev.ptr(self.d_segs), dev.ptr(self.d_chunks), chunk0, n,
                         1 if g_is_f16 else 0, dev.ptr(self.params), self.hint,
                         dev.ptr(self.partials), dev.ptr(self.flags), stream_h)

    def trust(self, stream_h: int, peer_flags: torch.Tensor | None = None, npeers: int = 0):
        _native.call("gs_lars_trust", dev.ptr(self.d_segs), self.nseg, dev.ptr(self.partials),
                     dev.ptr(self.params), dev.ptr(self.seg_scale), dev.ptr(self.seg_out),
                     dev.ptr(self.grad_norm), dev.ptr(self.counters[self.nseg:]),
                     dev.ptr(peer_flags) if peer_flags is not None else None, npeers,
                     dev.ptr(self.flags), stream_h)

    def pass2(self, stream_h: int, g_is_f16: bool, flag_mask: int, chunk0: int = 0,
              nchunk: int | None = None, trust: bool = False):
        """trust=True: gs_lars_pass2_trust (the trust ratio folded per CTA,
        no separate trust launch; needs pass 1 without fusion)."""
        n = self.nchunk - chunk0 if nchunk is None else nchunk
        if trust:
            _native.call("gs_lars_pass2_trust", dev.ptr(self.d_segs), self.nseg, self.nseg_active,
                         dev.ptr(self.d_chunks), chunk0, n, 1 if g_is_f16 else 0,
                         dev.ptr(self.params), self.hint, dev.ptr(self.partials),
                         dev.ptr(self.seg_scale), dev.ptr(self.seg_out), dev.ptr(self.grad_norm),
                         dev.ptr(self.counters[self.nseg:]), dev.ptr(self.flags), flag_mask,
                         stream_h)
            return
        _native.call("gs_lars_pass2", dev.ptr(self.d_segs), dev.ptr(self.d_chunks), chunk0, n,
                     1 if g_is_f16 else 0, dev.ptr(self.params), self.hint, dev.ptr(self.seg_scale),
                     dev.ptr(self.flags), flag_mask, stream_h)

    @property
    def trust_via_pass2(self) -> bool:
        return not self.fused and self.trust_in_pass2 and self.nseg_active > 0

    def finish(self, stream_h: int, g_is_f16: bool, flag_mask: int) -> None:
        """trust (unless pass 1 fused it) + pass 2, in the configured form."""
        if self.trust_via_pass2:
            self.pass2(stream_h, g_is_f16, flag_mask, trust=True)
            return
        if not self.fused:
            self.trust(stream_h)
        self.pass2(stream_h, g_is_f16, flag_mask)

    def run(self, stream_h: int, g_is_f16: bool, flag_mask: int) -> None:
        self.reset_flags(stream_h)
        self.pass1(stream_h, g_is_f16)
        self.finish(stream_h, g_is_f16, flag_mask)
