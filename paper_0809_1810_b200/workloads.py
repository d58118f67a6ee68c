"""Seeded synthetic particle sets for the BASELINE.json configurations.

SURVEY.md §8(d) defines them; BASELINE.json names no dataset, so these are the
inputs (no public suite is reproduced).  Domain is always [-1, 1]^2 passed
explicitly, kernel GAUSSIAN, uniform sigma; random draws use numpy PCG64 with
seed 1 and the draw order of the reference generator (model.py:102-109):
one (N, 2) uniform position draw, then the circulation draw.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

NU_T = 0.05  # Lamb-Oseen nu*t


@dataclass(frozen=True)
class Workload:
    name: str
    x: np.ndarray
    y: np.ndarray
    gamma: np.ndarray
    sigma: np.ndarray
    levels: int
    order: int

    @property
    def n(self) -> int:
        return int(self.x.size)


DOMAIN = (-1.0, -1.0, 2.0)  # (xmin, ymin, side)


def lamb_oseen(x: np.ndarray, y: np.ndarray, xc: float, yc: float) -> np.ndarray:
    """omega(x) = exp(-|x - x_c|^2 / (4 nu t)) / (4 pi nu t)."""
    r2 = (x - xc) ** 2 + (y - yc) ** 2
    return np.exp(-r2 / (4.0 * NU_T)) / (4.0 * np.pi * NU_T)


def lattice(m: int) -> tuple[np.ndarray, np.ndarray, float]:
    """Cell-centred m x m lattice over [-1, 1]^2, row-major via meshgrid(c, c)."""
    h = 2.0 / m
    c = -1.0 + (np.arange(m) + 0.5) * h
    gx, gy = np.meshgrid(c, c)
    return gx.ravel().copy(), gy.ravel().copy(), h


def uniform(n: int, seed: int = 1):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(size=(n, 2))
    return rng, -1.0 + 2.0 * pos[:, 0], -1.0 + 2.0 * pos[:, 1]


def config0(m: int = 64, levels: int = 3, order: int = 10) -> Workload:
    x, y, h = lattice(m)
    g = lamb_oseen(x, y, 0.0, 0.0) * h * h
    return Workload(f"config0_lattice{m}", x, y, g, np.full(x.size, h / 0.8), levels, order)


def config1(n: int = 65536, seed: int = 1) -> Workload:
    rng, x, y = uniform(n, seed)
    h = 2.0 / 256
    g = rng.standard_normal(n) * h * h
    return Workload("config1_uniform_normal", x, y, g, np.full(n, 1.25 * h), 5, 12)


def config2(m: int = 1024) -> Workload:
    x, y, h = lattice(m)
    g = (lamb_oseen(x, y, 0.0, 0.0) - lamb_oseen(x, y, 0.5, 0.0)) * h * h
    return Workload("config2_lattice_two_vortices", x, y, g, np.full(x.size, h / 0.8), 7, 17)


def config3(n: int = 1 << 24, seed: int = 1) -> Workload:
    rng, x, y = uniform(n, seed)
    h = 2.0 / 4096
    g = rng.uniform(-1.0, 1.0, n) * h * h
    return Workload("config3_uniform", x, y, g, np.full(n, 1.25 * h), 9, 20)


def config4(m: int, levels: int, order: int) -> Workload:
    """Error-study case: lattice Lamb-Oseen as config 0 at (m, levels, order)."""
    w = config0(m, levels, order)
    return Workload(f"config4_m{m}_l{levels}_p{order}", w.x, w.y, w.gamma, w.sigma, levels, order)


CONFIG4_GRID = [
    (m, lv, p) for m in (64, 128, 256, 512, 1024) for lv in range(3, 9) for p in (5, 10, 15, 20, 25)
]


def by_index(i: int) -> Workload:
    return (config0, config1, config2, config3)[i]()


def generate_particles(distribution: str, n: int, seed: int, domain=(0.0, 0.0, 1.0),
                       sigma: float = 0.005):
    """Seeded particle sets of the reference generator (model.py:71-122), as arrays.

    One (n, 2) uniform position draw, then the circulation draw:
    ``uniform_random`` Gamma ~ U(-1, 1); ``gaussian_patch`` Gamma =
    exp(-r^2 / (2 s^2)) side^2 / n about the centre, s = side / 8;
    ``two_patches`` the difference of two such patches at (1/4, 1/2) and
    (3/4, 1/2) of the domain.  Used by the acceptance tests that reproduce
    the reference's published numbers (test_output.txt:11-19).
    """
    xmin, ymin, side = domain
    rng = np.random.default_rng(seed)
    pos = rng.uniform(size=(n, 2))
    x = xmin + side * pos[:, 0]
    y = ymin + side * pos[:, 1]
    s = side / 8.0
    if distribution == "uniform_random":
        g = rng.uniform(-1.0, 1.0, n)
    elif distribution == "gaussian_patch":
        cx, cy = xmin + 0.5 * side, ymin + 0.5 * side
        g = np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2.0 * s * s)) * side**2 / n
    elif distribution == "two_patches":
        cy = ymin + 0.5 * side
        ra = (x - (xmin + 0.25 * side)) ** 2 + (y - cy) ** 2
        rb = (x - (xmin + 0.75 * side)) ** 2 + (y - cy) ** 2
        g = (np.exp(-ra / (2.0 * s * s)) - np.exp(-rb / (2.0 * s * s))) * side**2 / n
    else:
        raise ValueError(f"unknown distribution {distribution!r}")
    return x, y, g, np.full(n, float(sigma))
