"""Median per-phase times (stats mode with phase events, serialised phases) of
one BASELINE config: build / upward / m2l / downward (L2L + L2P + combine) /
near / total.  Usage: phase_probe.py [config] [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import workloads as W  # noqa: E402

cfg_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
w = W.by_index(cfg_idx)
dev = torch.device("cuda", 0)
xs, ys, gs, ss = w.x, w.y, w.gamma, w.sigma
if os.environ.get("PROBE_PRESORT"):  # the same particles in leaf order (a coherent input order)
    import numpy as np

    m = 1 << w.levels
    ix = np.minimum(((xs + 1.0) / 2.0 * m).astype(np.int64), m - 1)
    iy = np.minimum(((ys + 1.0) / 2.0 * m).astype(np.int64), m - 1)
    o = np.argsort(iy * m + ix, kind="stable")
    xs, ys, gs, ss = xs[o], ys[o], gs[o], ss[o]
xd, yd, gd, sd = (torch.from_numpy(a).to(dev) for a in (xs, ys, gs, ss))
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
keys = ("t_build", "t_upward", "t_m2l", "t_downward", "t_near", "t_total")
rows = {k: [] for k in keys}
for _ in range(reps):
    _, st = vf.evaluate_arrays(xd, yd, gd, sd, cfg, vf.Domain(*W.DOMAIN), timings=True)
    for k in keys:
        rows[k].append(getattr(st, k) * 1e3)
lib = os.environ.get("VFMM_LIB", "default")
print(f"{lib} {w.name}: " + "  ".join(f"{k[2:]} {statistics.median(v[2:]):.4f}" for k, v in rows.items()))
