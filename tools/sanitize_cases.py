"""Small evaluations that cover every kernel of libvfmm.so, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases (default: all):
  config0   lattice N=4096 l=3 p=10: counting sort, symmetric P2P, fused L2L+L2P
  overlap   config 0 with the near field on the side stream
  config1   uniform N=65536 l=5 p=12: random order -> LSD radix sort path
  generic   non-uniform sigma -> generic P2P (k_p2p, cp.async double buffer)
  bigleaf   a leaf > 128 particles -> LSD path + generic P2P
  graph     vfmm_evaluate_host with VFMM_FLAG_GRAPH (captured + replayed)
  direct    vfmm_direct (tiled O(N^2) kernel)
  at        vfmm_evaluate_at
  shard     two row strips through vfmm_evaluate_shard (PHASE_UP / PHASE_DOWN)
Each case also checks its result against the numpy oracle (test infrastructure).
"""

from __future__ import annotations

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from oracle import fmm_oracle as O  # noqa: E402
from paper_0809_1810_b200 import workloads as W  # noqa: E402

G = vf.KernelKind.GAUSSIAN_BLOB
DOM = vf.Domain(*W.DOMAIN)


def check(name, got, ref, tol=1e-12):
    err = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))
    print(f"{name}: max rel err {err:.2e}", flush=True)
    assert err <= tol, name


def run_eval(name, w, overlap=False):
    vel, st = vf.evaluate_arrays(w.x, w.y, w.gamma, w.sigma, vf.FmmConfig(w.levels, w.order, G), DOM,
                                 overlap=overlap)
    ref, _ = O.evaluate(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    check(name, vel.cpu().numpy().T, ref)


def case_config0():
    run_eval("config0", W.config0())


def case_overlap():
    run_eval("overlap", W.config0(), overlap=True)


def case_config1():
    run_eval("config1", W.config1())


def case_generic():
    w = W.config1(n=8192)
    s = w.sigma * (1.0 + 0.1 * np.random.default_rng(3).uniform(size=w.n))
    run_eval("generic", W.Workload("generic", w.x, w.y, w.gamma, s, 4, 10))


def case_bigleaf():
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-0.1, -0.05, 300), rng.uniform(-1, 1, 2000)])
    y = np.concatenate([rng.uniform(0.2, 0.25, 300), rng.uniform(-1, 1, 2000)])
    g = rng.uniform(-1, 1, x.size) * 1e-3
    run_eval("bigleaf", W.Workload("bigleaf", x, y, g, np.full(x.size, 0.004), 4, 8))


def case_graph():
    w = W.config0()
    cfg = vf.FmmConfig(w.levels, w.order, G)
    ref, _ = O.evaluate(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    for _ in range(2):  # capture, then replay
        out, _ = vf.evaluate_host(w.x, w.y, w.gamma, w.sigma, cfg, DOM, graph=True)
        check("graph", out.numpy(), ref)


def case_direct():
    w = W.config1(n=4096)
    u, v = vf.velocity_direct_arrays(w.x, w.y, w.x, w.y, w.gamma, w.sigma, G)
    ref = O.direct(w.x, w.y, w.x, w.y, w.gamma, w.sigma, True)
    check("direct", np.stack((u.cpu().numpy(), v.cpu().numpy()), axis=1), ref, 1e-13)


def case_at():
    w = W.config0()
    tx = np.linspace(-0.95, 0.95, 257)
    ty = np.linspace(0.9, -0.9, 257)
    cfg = vf.FmmConfig(w.levels, w.order, G)
    u, v = vf.evaluate_at_arrays(tx, ty, w.x, w.y, w.gamma, w.sigma, cfg, DOM)
    ref = O.evaluate_at(tx, ty, w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    check("at", np.stack((u.cpu().numpy(), v.cpu().numpy()), axis=1), np.asarray(ref).reshape(-1, 2))


def case_shard():
    from paper_0809_1810_b200 import distributed as D

    w = W.config0()
    ref, _ = O.evaluate(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    t = [torch.as_tensor(a, device="cuda") for a in (w.x, w.y, w.gamma, w.sigma)]
    vel, _, _ = D.evaluate_emulated(*t, vf.FmmConfig(w.levels, w.order, G), DOM, 2)
    check("shard", vel.cpu().numpy().T, ref)


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
    torch.cuda.synchronize()
    print("sanitize cases done:", " ".join(names))
