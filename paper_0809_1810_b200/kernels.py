"""Kernel kinds and the O(N^2) direct sum (north-star item 6) on the GPU.

Mirrors ``vortexfmm.kernels`` (reference ``kernels.py:24-94``):
``KernelKind`` has the same members and values, ``velocity_direct`` has the
same signature and returns an (M, 2) float64 array of (u, v) rows.  The sum
runs in the CUDA kernel ``k_direct`` (``csrc/p2p.cu``) via ``vfmm_direct``.
"""

from __future__ import annotations

import ctypes
import enum
import math
from typing import Sequence

import numpy as np

from . import _lib
from ._device import as_device_f64, device_of, require_cuda, stream_ptr, torch

TWO_PI = 2.0 * math.pi


class KernelKind(enum.Enum):
    """kernels.py:27-29."""

    POINT_VORTEX = "point_vortex"
    GAUSSIAN_BLOB = "gaussian_blob"


def kernel_code(kind) -> int:
    """C-ABI kernel code for our or the reference's KernelKind (matched by value)."""
    value = getattr(kind, "value", kind)
    if value == KernelKind.POINT_VORTEX.value:
        return _lib.KERNEL_POINT
    if value == KernelKind.GAUSSIAN_BLOB.value:
        return _lib.KERNEL_GAUSSIAN
    raise ValueError(f"unknown kernel kind {kind!r}")


def velocity_direct_arrays(tx, ty, x, y, gamma, sigma, kind, device=None):
    """Direct sum on device tensors; returns (u, v) float64 CUDA tensors of length M."""
    require_cuda()
    lib = _lib.load()
    dev = device_of(device, tx, x)
    tx, ty = as_device_f64(tx, dev), as_device_f64(ty, dev)
    m = int(tx.numel())
    n = int(torch.as_tensor(x).numel())
    u = torch.empty(m, dtype=torch.float64, device=dev)
    v = torch.empty(m, dtype=torch.float64, device=dev)
    if m == 0:
        return u, v
    if n == 0:
        u.zero_()
        v.zero_()
        return u, v
    x, y, gamma = (as_device_f64(a, dev) for a in (x, y, gamma))
    code = kernel_code(kind)
    sigma = as_device_f64(sigma, dev) if code == _lib.KERNEL_GAUSSIAN else None
    need = ctypes.c_size_t()
    _lib.check(lib.vfmm_direct_workspace_size(m, n, ctypes.byref(need)), "vfmm_direct_workspace_size")
    ws = torch.empty(max(int(need.value), 8), dtype=torch.uint8, device=dev)
    st = lib.vfmm_direct(
        tx.data_ptr(), ty.data_ptr(), m, x.data_ptr(), y.data_ptr(), gamma.data_ptr(),
        sigma.data_ptr() if sigma is not None else None, n, code, u.data_ptr(), v.data_ptr(),
        ws.data_ptr(), ws.numel(), stream_ptr(dev),
    )
    _lib.check(st, "vfmm_direct")
    return u, v


def velocity_direct(targets, sources: Sequence, kind) -> np.ndarray:
    """Direct summation over all sources at each target (kernels.py:52-94)."""
    from .model import to_arrays

    pts = np.asarray(targets, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 2:
        raise ValueError(f"targets must have shape (M, 2), got {pts.shape}")
    x, y, gamma, sigma = to_arrays(sources)
    u, v = velocity_direct_arrays(
        np.ascontiguousarray(pts[:, 0]), np.ascontiguousarray(pts[:, 1]), x, y, gamma, sigma, kind
    )
    return torch.stack((u, v), dim=1).cpu().numpy()
