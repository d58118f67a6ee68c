import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_0809_1810_b200 as vf
from paper_0809_1810_b200 import workloads as W
w = W.by_index(3)
dev = torch.device("cuda", 0)
xd, yd, gd, sd = (torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
for _ in range(2):
    vf.evaluate_arrays(xd, yd, gd, sd, cfg, vf.Domain(*W.DOMAIN))
torch.cuda.synchronize()
