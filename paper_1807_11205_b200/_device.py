"""Device-side plumbing shared by the drop-in modules.

PyTorch is used only for device memory and streams: arrays handed to the
reference-shaped API may be numpy arrays (they are moved to the GPU, the
result comes back as numpy, mirroring the reference's numpy-in/numpy-out
contract) or CUDA tensors (results stay on the device).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native

_NP_TO_TORCH = {
    np.dtype(np.float32): torch.float32,
    np.dtype(np.uint16): torch.uint16,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.uint8): torch.uint8,
}
_TORCH_TO_NP = {v: k for k, v in _NP_TO_TORCH.items()}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "a CUDA device is required: gradsync_b200 runs its arithmetic only in "
            "libgradsync_b200 kernels and has no CPU fallback")
    _native.lib()
    return torch.device("cuda", torch.cuda.current_device())


def is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def np_dtype_of(t: torch.Tensor) -> np.dtype:
    return _TORCH_TO_NP[t.dtype]


def torch_dtype(dt) -> torch.dtype:
    if isinstance(dt, torch.dtype):
        return dt
    return _NP_TO_TORCH[np.dtype(dt)]


def to_cuda(x, device: torch.device | None = None) -> torch.Tensor:
    """numpy array / CUDA tensor -> contiguous CUDA tensor (copy only if needed)."""
    dev = device or require_cuda()
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(dev)
    else:
        a = np.ascontiguousarray(x)
        t = torch.from_numpy(a).to(dev)
    return t.contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def upload(table: np.ndarray, device: torch.device, stream=None) -> torch.Tensor:
    """Copy a host struct table to device memory (returned tensor owns it)."""
    raw = np.ascontiguousarray(table).view(np.uint8).reshape(-1)
    host = torch.from_numpy(raw.copy()).pin_memory() if torch.cuda.is_available() else torch.from_numpy(raw.copy())
    dev = torch.empty(host.numel(), dtype=torch.uint8, device=device)
    if stream is None:
        dev.copy_(host, non_blocking=True)
    else:
        with torch.cuda.stream(stream):
            dev.copy_(host, non_blocking=True)
    # keep the pinned staging buffer alive until the copy has run
    dev._gs_host_stage = host  # type: ignore[attr-defined]
    return dev


def ptr(t: torch.Tensor) -> int:
    return int(t.data_ptr())


def stream_of(stream=None) -> int:
    return _native.stream_handle(stream)
