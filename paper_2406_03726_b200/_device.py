"""Device plumbing: PyTorch owns device memory and streams; libgee computes."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import GpuUnavailableError


def require_gpu() -> torch.device:
    if not torch.cuda.is_available():
        raise GpuUnavailableError("no CUDA device visible; this package has no CPU path")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if t.numel() > 0 else None


_NP_TO_TORCH = {
    np.dtype(np.int64): torch.int64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.uint32): torch.int32,
}


def to_device(x, dtype: torch.dtype, dev: torch.device) -> torch.Tensor:
    """numpy / torch -> contiguous device tensor of `dtype` (no copy if already so)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.device != dev:
            t = t.to(dev, non_blocking=True)
        if t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    a = np.ascontiguousarray(x)
    t = torch.from_numpy(a) if a.dtype in _NP_TO_TORCH else torch.as_tensor(a)
    if t.is_pinned():
        t = t.to(dev, non_blocking=True)
    else:
        t = t.to(dev)
    return t.to(dtype) if t.dtype != dtype else t


class Workspace:
    """Grow-only per-device scratch buffer (CUB-style size query, then reuse)."""

    def __init__(self):
        self._buf = {}

    def get(self, nbytes: int, dev: torch.device) -> torch.Tensor:
        key = dev.index
        buf = self._buf.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
            self._buf[key] = buf
        return buf


WORKSPACE = Workspace()


def error_word(dev: torch.device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=dev)


def check_device_errors(err: torch.Tensor, context: str = ""):
    _lib.raise_device_errors(int(err.item()), context)
