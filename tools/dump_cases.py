"""Velocities of a fixed set of evaluations saved to an .npz (argv[1]), for
bitwise comparisons between builds of libvfmm.so (VFMM_LIB): the plain build
vs the jittered one (tests/test_checked_build.py).  Covers the counting and
LSD sort paths, the symmetric (split and unsplit) and generic near fields, the
tiled and direct M2L kernels, graph replay and the sharded exchange."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import distributed as D, workloads as W  # noqa: E402

G = vf.KernelKind.GAUSSIAN_BLOB
DOM = vf.Domain(*W.DOMAIN)
out = {}
torch.cuda.set_device(0)


def ev(name, w, **kw):
    vel, st = vf.evaluate_arrays(w.x, w.y, w.gamma, w.sigma, vf.FmmConfig(w.levels, w.order, G), DOM, **kw)
    out[name] = vel.cpu().numpy()
    out[name + "_counts"] = np.array([st.m2l_count, st.near_pair_count])


ev("config0", W.config0())
ev("config0_overlap", W.config0(), overlap=True)
ev("config1", W.config1())
ev("config2", W.config2(), overlap=True)
w = W.config1(n=8192)
s = w.sigma * (1.0 + 0.1 * np.random.default_rng(3).uniform(size=w.n))
ev("generic", W.Workload("generic", w.x, w.y, w.gamma, s, 4, 10))
w2 = W.config0()
hv, _ = vf.evaluate_host(w2.x, w2.y, w2.gamma, w2.sigma, vf.FmmConfig(3, 10, G), DOM, graph=True)
hv, _ = vf.evaluate_host(w2.x, w2.y, w2.gamma, w2.sigma, vf.FmmConfig(3, 10, G), DOM, graph=True)
hv, _ = vf.evaluate_host(w2.x, w2.y, w2.gamma, w2.sigma, vf.FmmConfig(3, 10, G), DOM, graph=True)
out["graph"] = hv.numpy().copy()
w1 = W.config1()
t = [torch.from_numpy(a).cuda() for a in (w1.x, w1.y, w1.gamma, w1.sigma)]
vel, m2l, near = D.evaluate_emulated(*t, vf.FmmConfig(w1.levels, w1.order, G), DOM, 4)
out["shard4"] = vel.cpu().numpy()
np.savez(sys.argv[1], **out)
print("dumped", len(out), "arrays to", sys.argv[1])
