import sys, torch
sys.path.insert(0,'.')
import paper_0809_1810_b200 as vf
from paper_0809_1810_b200 import workloads as W
w = W.by_index(int(sys.argv[1]) if len(sys.argv) > 1 else 2); dev = torch.device('cuda',0)
t = [torch.from_numpy(a).to(dev) for a in (w.x,w.y,w.gamma,w.sigma)]
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
for i in range(4):
    vf.evaluate_arrays(*t, cfg, vf.Domain(*W.DOMAIN), overlap=True, timings=True)
