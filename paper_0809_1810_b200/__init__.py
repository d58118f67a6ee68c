"""B200-native FMM velocity evaluation for 2-D Gaussian-regularised vortex
particles (arXiv 0809.1810), a drop-in for the hot path of the reference
package ``vortexfmm`` (``engine.evaluate``, ``engine.py:335-398``).

The public names mirror ``vortexfmm/__init__.py:9-20`` for the hot path:
``evaluate``, ``evaluate_at``, ``FmmConfig``, ``FmmRunStats``, ``KernelKind``,
``velocity_direct``, ``Particle``, ``Domain``.  All compute runs in the
hand-written sm_100a CUDA library ``libvfmm.so`` (C ABI: ``include/vfmm.h``).
"""

from . import errors
from .engine import (
    FmmConfig,
    FmmRunStats,
    HostPipeline,
    PendingEvaluation,
    Workspace,
    evaluate,
    evaluate_arrays,
    evaluate_at,
    evaluate_at_arrays,
    evaluate_host,
    evaluate_host_async,
)
from .kernels import TWO_PI, KernelKind, velocity_direct, velocity_direct_arrays
from .model import Domain, Particle, enclosing_domain, to_arrays
from .quadtree import OutOfDomainError, grid_indices

__version__ = "0.1.0"

__all__ = [
    "Domain",
    "errors",
    "FmmConfig",
    "FmmRunStats",
    "HostPipeline",
    "KernelKind",
    "OutOfDomainError",
    "Particle",
    "PendingEvaluation",
    "TWO_PI",
    "Workspace",
    "enclosing_domain",
    "evaluate",
    "evaluate_arrays",
    "evaluate_at",
    "evaluate_at_arrays",
    "evaluate_host",
    "evaluate_host_async",
    "grid_indices",
    "to_arrays",
    "velocity_direct",
    "velocity_direct_arrays",
]
