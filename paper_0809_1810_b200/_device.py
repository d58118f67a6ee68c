"""Device plumbing shared by the host modules: torch tensors for device memory,
the caller's current CUDA stream, and loud failure when CUDA is unavailable."""

from __future__ import annotations

import numpy as np
import torch


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_0809_1810_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback"
        )


def device_of(device=None, *tensors) -> torch.device:
    if device is not None:
        return torch.device(device)
    for t in tensors:
        if isinstance(t, torch.Tensor) and t.is_cuda:
            return t.device
    return torch.device("cuda", torch.cuda.current_device())


def as_device_f64(a, dev: torch.device) -> torch.Tensor:
    """float64 contiguous CUDA tensor view/copy of a numpy array or tensor."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    if t.dtype != torch.float64:
        t = t.to(torch.float64)
    if t.device != dev:
        t = t.to(dev, non_blocking=t.is_pinned())
    return t.contiguous()


def stream_ptr(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream
