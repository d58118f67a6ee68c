"""Run a few full evaluates of one BASELINE config (default 2) for ncu / sanitizer captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import workloads as W  # noqa: E402

cfg_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = W.by_index(cfg_idx)
dev = torch.device("cuda", 0)
xd, yd, gd, sd = (torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
for _ in range(reps):
    vel, st = vf.evaluate_arrays(xd, yd, gd, sd, cfg, vf.Domain(*W.DOMAIN))
torch.cuda.synchronize()
print(f"{w.name}: t_total={st.t_total * 1e3:.3f} ms near={st.t_near * 1e3:.3f} ms m2l={st.t_m2l * 1e3:.3f} ms")
