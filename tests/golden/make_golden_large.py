"""Generate the LARGE golden vectors by running the REFERENCE implementation.

Companion of ``make_golden.py`` for the full-size BASELINE configurations and
the config-4 error study at N >= 2^16.  Run in the build container, where the
reference is mounted read-only (needs ~12 GB of RAM and ~15 min on 8 cores):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_large.py

Nothing is copied from the reference: it is imported from
/root/reference/pkg/src and only its OUTPUTS are stored, in
``tests/golden/golden_large.npz``:

* ``full/config2`` and ``full/config3`` -- ``vortexfmm.engine.evaluate`` on
  the full BASELINE config 2 (N = 2^20, l = 7, p = 17) and config 3
  (N = 2^24, l = 9, p = 20), GAUSSIAN, Domain(-1, -1, 2): an input digest,
  the exact counters, max|v| over ALL particles, the column sums of (u, v)
  and the velocities at 65,536 seeded sample indices (engine.py:335-398).
* ``map16/<l>_<p>`` -- config 4 at N = 2^16 (m = 256): the reference FMM vs
  the reference ``velocity_direct`` over all N targets, reduced to the
  errors.compare scalars and errors.spatial_map maps at g = 8 and g = 32
  (errors.py:46-120), plus the per-target direct velocities (once per N).
* ``samp/<m>_<l>_<p>`` -- config 4 at N = 2^18 and 2^20 (l >= 5): reference
  FMM velocities and reference direct velocities at the harness's sampled
  targets (``default_rng([seed, n, l, p, 0x0F5EED])``, k = 256,
  harness.py:235-245) and the exact counters.

The GPU box never needs the reference: tests read only the .npz.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time
import warnings

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

SAMPLE_SEED = 20261020
N_SAMPLE = 65536
HARNESS_SEED = 1
HARNESS_K = 256
MAP16 = [(3, 5), (4, 10), (5, 15), (6, 20), (7, 25), (8, 10)]
SAMPLED = [(512, 5, 5), (512, 6, 10), (512, 7, 15), (512, 8, 20),
           (1024, 5, 10), (1024, 6, 15), (1024, 7, 20), (1024, 8, 25)]


def digest(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()[:16]


def particles(x, y, g, s):
    from vortexfmm.model import Particle

    return [Particle(float(a), float(b), float(c), float(d)) for a, b, c, d in zip(x, y, g, s)]


def ref_eval(w, levels, order):
    import vortexfmm as ref
    from vortexfmm.engine import FmmConfig
    from vortexfmm.kernels import KernelKind
    from vortexfmm.model import Domain

    parts = particles(w.x, w.y, w.gamma, w.sigma)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        vel, st = ref.evaluate(parts, FmmConfig(levels, order, KernelKind.GAUSSIAN_BLOB),
                               Domain(-1.0, -1.0, 2.0))
    return parts, vel, st


def job_full(idx: int):
    from paper_0809_1810_b200 import workloads as W

    w = W.by_index(idx)
    t0 = time.perf_counter()
    _, vel, st = ref_eval(w, w.levels, w.order)
    wall = time.perf_counter() - t0
    sample = np.sort(np.random.default_rng(SAMPLE_SEED).choice(w.n, N_SAMPLE, replace=False))
    pre = f"full/config{idx}/"
    return {
        pre + "digest": np.array(digest(w.x, w.y, w.gamma, w.sigma)),
        pre + "cfg": np.array([w.n, w.levels, w.order]),
        pre + "counts": np.array([st.m2l_count, st.near_pair_count, int(st.sigma_guard_ok)]),
        pre + "vmax": np.array(np.abs(vel).max()),
        pre + "speed_max": np.array(np.hypot(vel[:, 0], vel[:, 1]).max()),
        pre + "colsum": vel.sum(axis=0),
        pre + "sample": sample,
        pre + "vel": vel[sample],
        pre + "ref_t_total": np.array(st.t_total),
        pre + "ref_wall": np.array(wall),
    }


def job_map16():
    import vortexfmm as ref
    from vortexfmm import errors as E
    from vortexfmm.engine import bound_budgets
    from vortexfmm.kernels import KernelKind
    from vortexfmm.model import Domain
    from vortexfmm.quadtree import build_tree

    from paper_0809_1810_b200 import workloads as W

    out = {}
    w = W.config4(256, 3, 5)
    parts = particles(w.x, w.y, w.gamma, w.sigma)
    pos = np.stack((w.x, w.y), axis=1)
    t0 = time.perf_counter()
    direct = ref.velocity_direct(pos, parts, KernelKind.GAUSSIAN_BLOB)
    out["map16/direct_seconds"] = np.array(time.perf_counter() - t0)
    out["map16/direct"] = direct
    box = Domain(-1.0, -1.0, 2.0)
    for lv, p in MAP16:
        _, vel, st = ref_eval(w, lv, p)
        bud = bound_budgets(build_tree(parts, lv, box), w.gamma, p)
        rep = E.compare(vel, direct, pos, bud)
        pre = f"map16/{lv}_{p}/"
        out[pre + "counts"] = np.array([st.m2l_count, st.near_pair_count, int(st.sigma_guard_ok)])
        out[pre + "scalars"] = np.array([rep.max_abs, rep.max_rel, rep.rms_abs, rep.rms_rel])
        out[pre + "violations"] = np.array(len(E.bound_check(rep)))
        out[pre + "vel_sample"] = vel[:: 97]
        for g in (8, 32):
            em = E.spatial_map(rep, box, g)
            out[pre + f"map{g}_counts"] = em.counts
            out[pre + f"map{g}_max"] = em.max_err
            out[pre + f"map{g}_mean"] = em.mean_err
    return out


def job_sampled(m: int, lv: int, p: int):
    import vortexfmm as ref
    from vortexfmm.kernels import KernelKind

    from paper_0809_1810_b200 import workloads as W

    w = W.config4(m, lv, p)
    n = w.n
    parts, vel, st = ref_eval(w, lv, p)
    rng = np.random.default_rng([HARNESS_SEED, n, lv, p, 0x0F5EED])
    sample = np.sort(rng.choice(n, size=HARNESS_K, replace=False))
    pos = np.stack((w.x, w.y), axis=1)
    direct = ref.velocity_direct(pos[sample], parts, KernelKind.GAUSSIAN_BLOB)
    pre = f"samp/{m}_{lv}_{p}/"
    return {
        pre + "counts": np.array([st.m2l_count, st.near_pair_count, int(st.sigma_guard_ok)]),
        pre + "sample": sample,
        pre + "fmm": vel[sample],
        pre + "direct": direct,
        pre + "vmax_fmm": np.array(np.abs(vel).max()),
    }


def run(job):
    kind, args = job
    t0 = time.perf_counter()
    res = {"full": job_full, "map16": job_map16, "sampled": job_sampled}[kind](*args)
    print(f"  {kind}{args}: {time.perf_counter() - t0:.1f} s", flush=True)
    return res


def main():
    import multiprocessing as mp

    jobs = [("full", (3,)), ("map16", ()), ("full", (2,))] + [("sampled", c) for c in SAMPLED]
    out: dict[str, np.ndarray] = {}
    with mp.get_context("fork").Pool(int(os.environ.get("GOLDEN_PROCS", "6"))) as pool:
        for res in pool.imap_unordered(run, jobs):
            out.update(res)
    out["meta/sample_seed"] = np.array(SAMPLE_SEED)
    out["meta/map16_cases"] = np.array([f"{lv}_{p}" for lv, p in MAP16])
    out["meta/sampled_cases"] = np.array([f"{m}_{lv}_{p}" for m, lv, p in SAMPLED])
    path = os.path.join(HERE, "golden_large.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
