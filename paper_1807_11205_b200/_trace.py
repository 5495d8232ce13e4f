"""NVTX phase ranges of the pipeline's host-side launch sequence.

Enabled with ``GS_NVTX=1`` (or ``set_enabled(True)``): every phase the
pipeline reports to its timer hook (pack, all-reduce of bucket b, pass 1,
trust, pass 2, the fused reduce-scatter + pass 1 ...) becomes an NVTX range
``gs.<phase>`` on the launching thread and a ``record_function`` range in a
torch.profiler trace, nested in one ``gs.step`` range, so an nsys / Kineto
timeline shows which launch belongs to which phase next to the kernels.
Disabled, the hook is absent and the launch path does no work for it.
"""

from __future__ import annotations

import os

import torch

_enabled = os.environ.get("GS_NVTX", "0") == "1"


def set_enabled(on: bool) -> None:
    global _enabled
    _enabled = bool(on)


def enabled() -> bool:
    return _enabled


class PhaseRanges:
    """A timer hook that closes the previous phase range and opens the next;
    chains to an inner hook (the bench's CUDA-event timer)."""

    def __init__(self, inner=None, outer: str = "gs.step"):
        self.inner = inner
        self.open = None
        self._outer = torch.profiler.record_function(outer)
        self._outer.__enter__()
        torch.cuda.nvtx.range_push(outer)

    def __call__(self, name: str) -> None:
        if self.inner is not None:
            self.inner(name)
        self._close()
        if name != "end":
            self.open = torch.profiler.record_function("gs." + name)
            self.open.__enter__()
            torch.cuda.nvtx.range_push("gs." + name)

    def _close(self) -> None:
        if self.open is not None:
            torch.cuda.nvtx.range_pop()
            self.open.__exit__(None, None, None)
            self.open = None

    def close(self) -> None:
        self._close()
        torch.cuda.nvtx.range_pop()
        self._outer.__exit__(None, None, None)


def hook(timer, outer: str = "gs.step"):
    """The timer hook a step uses: the caller's timer, wrapped in NVTX phase
    ranges when enabled."""
    return PhaseRanges(timer, outer) if _enabled else timer
