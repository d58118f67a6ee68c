"""Loader for tests/golden/golden.npz (generated from the reference by make_golden.py)."""
import hashlib
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = dict(np.load(os.path.join(HERE, "golden", "golden.npz"), allow_pickle=False))
CASES = [str(c) for c in GOLDEN["cases"]]
DIRECT_CASES = sorted({k.split("/")[1] for k in GOLDEN if k.startswith("direct/")})


def digest(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()[:16]


def eval_case(name):
    from paper_0809_1810_b200 import workloads as W

    G = GOLDEN
    pre = f"eval/{name}/"
    if pre + "x" in G:
        x, y, g, s = (G[pre + k] for k in ("x", "y", "gamma", "sigma"))
    else:
        w = W.config0() if name == "config0" else W.config1()
        x, y, g, s = w.x, w.y, w.gamma, w.sigma
    levels, order, gauss = (int(v) for v in G[pre + "cfg"])
    dom = G[pre + "domain"]
    domain = None if np.isnan(dom).any() else tuple(float(v) for v in dom)
    return dict(
        name=name, x=x, y=y, gamma=g, sigma=s, levels=levels, order=order, gauss=bool(gauss),
        domain=domain, m2l_count=int(G[pre + "counts"][0]), near_pair_count=int(G[pre + "counts"][1]),
        sigma_guard_ok=bool(G[pre + "counts"][2]), vel=G[pre + "vel"], vmax=float(G[pre + "vmax"]),
        sample=G.get(pre + "sample"), digest=str(G[pre + "digest"]),
    )


def enclosing(x, y):
    xmin, ymin = float(x.min()), float(y.min())
    side = float(max(x.max() - xmin, y.max() - ymin))
    return (xmin, ymin, side if side > 0 else 1.0)
