"""Quadtree vocabulary of the drop-in API.

The tree itself is built on the GPU (``csrc/tree.cu``); this module keeps the
reference's exception type and the floor-rule binning expression used on the
host (error maps, target checks): ``quadtree.py:19-20,39-46``.
"""

from __future__ import annotations

import numpy as np


class OutOfDomainError(ValueError):
    """A position (or particle) lies outside the domain square (quadtree.py:19-20)."""


def grid_indices(x, y, cells_per_side: int, domain) -> tuple[np.ndarray, np.ndarray]:
    """Floor-rule bin indices with max-edge clamp (quadtree.py:39-46)."""
    m = cells_per_side
    ix = np.minimum(((np.asarray(x) - domain.xmin) / domain.side * m).astype(np.int64), m - 1)
    iy = np.minimum(((np.asarray(y) - domain.ymin) / domain.side * m).astype(np.int64), m - 1)
    return ix, iy
