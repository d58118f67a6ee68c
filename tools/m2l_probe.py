"""M2L probe: median t_m2l (stats mode, serialised phases) on one BASELINE config,
its algorithmic TFLOP/s (8 (p+1)^2 flop per translation) and a
checksum of the velocities.  Run once per variant (the library reads its A/B
switches once per process), e.g. VFMM_M2L_TILE=0 for the direct-load kernel.
Usage: m2l_probe.py [config] [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import workloads as W  # noqa: E402

cfg_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
w = W.by_index(cfg_idx)
dev = torch.device("cuda", 0)
xd, yd, gd, sd = (torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
ts = []
for _ in range(reps):
    vel, st = vf.evaluate_arrays(xd, yd, gd, sd, cfg, vf.Domain(*W.DOMAIN), timings=True)
    ts.append(st.t_m2l * 1e3)
t = statistics.median(ts[2:])
flop = 8 * (w.order + 1) ** 2 * st.m2l_count
v = vel.cpu().numpy()
tag = "tile" if os.environ.get("VFMM_M2L_TILE", "1") != "0" else "direct"
print(f"{tag} {w.name}: m2l {t:.4f} ms ({flop / t / 1e9:.2f} TF/s algorithmic), m2l_count {st.m2l_count}, "
      f"checksum {np.abs(v).sum():.15e}")
