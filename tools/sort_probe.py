"""Build time of the counting path vs the LSD radix path on random-order
inputs of several sizes (stats mode, phase events).  Usage: sort_probe.py"""
import os
import statistics
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, statistics, numpy as np, torch
sys.path.insert(0, %r)
import paper_0809_1810_b200 as vf
n, levels = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(5)
x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
g = rng.normal(size=n); s = np.full(n, 2.0 / (1 << levels) / 8)
dev = torch.device("cuda", 0)
t = [torch.from_numpy(a).to(dev) for a in (x, y, g, s)]
cfg = vf.FmmConfig(levels, 10, vf.KernelKind.GAUSSIAN_BLOB)
b = []
for _ in range(7):
    _, st = vf.evaluate_arrays(*t, cfg, vf.Domain(-1.0, -1.0, 2.0), timings=True)
    b.append(st.t_build * 1e3)
print(statistics.median(b[2:]))
''' % REPO
for n, lv in ((1 << 20, 7), (1 << 21, 7), (1 << 22, 8), (1 << 23, 8), (1 << 24, 9)):
    res = {}
    for mode in ("count", "lsd"):
        out = subprocess.run([sys.executable, "-c", CODE, str(n), str(lv)], capture_output=True, text=True,
                             env=dict(os.environ, VFMM_SORT=mode))
        res[mode] = out.stdout.strip() or out.stderr[-200:]
    print(f"n = {n:>9} levels {lv}: build ms counting {res['count']}  lsd {res['lsd']}", flush=True)
