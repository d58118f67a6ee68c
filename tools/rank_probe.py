import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_0809_1810_b200 as vf
from paper_0809_1810_b200 import distributed as D, workloads as W
w = W.by_index(int(sys.argv[1])); world = int(sys.argv[2]); r = int(sys.argv[3])
dev = torch.device("cuda", 0)
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB); dom = vf.Domain(*W.DOMAIN)
x, y, g, s = (torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
sh = D.make_shards(x, y, g, s, dom, cfg.levels, world)[r]
be = D.CudaShardBackend(dev, private_workspace=True)
for _ in range(2):
    be.up(sh, cfg, dom); be.down(sh, cfg, dom, counters=False)
torch.cuda.synchronize()
