import sys; sys.path.insert(0, ".")
import numpy as np, paper_0809_1810_b200 as vf
from oracle import fmm_oracle as O
from paper_0809_1810_b200 import workloads as W
for idx in (0, 1):
    w = W.by_index(idx); cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
    v, st = vf.evaluate_arrays(w.x, w.y, w.gamma, w.sigma, cfg, vf.Domain(*W.DOMAIN)); v = v.cpu().numpy().T
    r, o = O.evaluate(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    print(w.name, "vs oracle", np.abs(v - r).max() / np.abs(r).max(), st.m2l_count, o["m2l_count"])
