"""Evaluate one BASELINE config (argv[1]) through a chosen path and save the
velocities at the golden sample indices + the counters to argv[2] (.npz);
the library's A/B switches (VFMM_SORT=lsd, VFMM_P2P_SYM=0, ...) are read once
per process, so tests/test_large_parity.py runs each variant in its own
process.  argv[3] (optional): "host_graph" (the public host-buffer API with
cached graph replay) or "sharded8" (8 logical ranks of the sharded path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import distributed as D, workloads as W  # noqa: E402

idx, path = int(sys.argv[1]), sys.argv[2]
mode = sys.argv[3] if len(sys.argv) > 3 else "device"
sample = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                              "golden_large.npz"))[f"full/config{idx}/sample"]
w = W.by_index(idx)
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
dom = vf.Domain(*W.DOMAIN)
torch.cuda.set_device(0)
if mode == "host_graph":
    for _ in range(3):  # stream call, capture, replay
        vel, st = vf.evaluate_host(w.x, w.y, w.gamma, w.sigma, cfg, dom, graph=True)
    v = vel.numpy()
    counts = (st.m2l_count, st.near_pair_count)
elif mode == "sharded8":
    t = [torch.from_numpy(a).cuda() for a in (w.x, w.y, w.gamma, w.sigma)]
    vel, m2l, near = D.evaluate_emulated(*t, cfg, dom, 8)
    v = vel.cpu().numpy().T
    counts = (m2l, near)
else:
    t = [torch.from_numpy(a).cuda() for a in (w.x, w.y, w.gamma, w.sigma)]
    vel, st = vf.evaluate_arrays(*t, cfg, dom, overlap=True)
    v = vel.cpu().numpy().T
    counts = (st.m2l_count, st.near_pair_count)
np.savez(path, vel=v[sample], vmax=np.abs(v).max(), counts=np.array(counts))
print("saved", path, counts)
