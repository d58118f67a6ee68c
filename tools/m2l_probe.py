"""M2L variant probe: median t_m2l (stats mode, serialised phases) of the
factored kernel vs the Hankel-row kernel (VFMM_M2L_HANKEL=1) on one BASELINE
config, and the max relative velocity difference between the two."""
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


def run(hankel):
    if hankel:
        os.environ["VFMM_M2L_HANKEL"] = "1"
    else:
        os.environ.pop("VFMM_M2L_HANKEL", None)
    ts = []
    for _ in range(reps):
        vel, st = vf.evaluate_arrays(xd, yd, gd, sd, cfg, vf.Domain(*W.DOMAIN), timings=True)
        ts.append(st.t_m2l * 1e3)
    torch.cuda.synchronize()
    return vel.cpu().numpy(), statistics.median(ts[2:]), st


vh, th, sh = run(True)
vfac, tf, sf = run(False)
err = float(np.abs(vfac - vh).max() / np.abs(vh).max())
flop = 8 * (w.order + 1) ** 2 * sf.m2l_count
print(f"{os.environ.get('VFMM_LIB', 'default')} {w.name}: m2l hankel {th:.4f} ms, factored {tf:.4f} ms "
      f"({flop / tf / 1e9:.2f} TF/s algorithmic), max rel diff {err:.2e}, counts {sh.m2l_count} {sf.m2l_count}")
