"""Where HostPipeline's host time goes: the pipeline as is, then with the
uniform-sigma check replaced by a constant.  Usage: e2e_host_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import engine as E, workloads as W  # noqa: E402

w = W.by_index(2)
dev = torch.device("cuda", 0)
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
dom = vf.Domain(*W.DOMAIN)
hx, hy, hg, hs = (torch.from_numpy(a).pin_memory() for a in (w.x, w.y, w.gamma, w.sigma))
orig = E._uniform_sigma
print("torch threads", torch.get_num_threads())


def run(p, steps=64):
    torch.cuda.synchronize()
    host = 0.0
    t0 = time.perf_counter()
    for _ in range(steps):
        i = p.k % len(p.slots)
        if p.pending[i] is not None:
            p.pending[i].wait()
        t1 = time.perf_counter()
        p.submit(hx, hy, hg, hs)
        host += time.perf_counter() - t1
    for q in p.pending:
        q.result()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / steps, host * 1e3 / steps


for d, c in ((4, 0), (4, 4), (8, 4)):
    p = vf.HostPipeline(w.n, cfg, dom, depth=d, device=dev, compute_streams=c)
    for mode in ("as is", "constant sigma check", "as is, 1 torch thread"):
        E._uniform_sigma = (lambda k: float(w.sigma[0])) if mode.startswith("constant") else orig
        torch.set_num_threads(1 if "1 torch" in mode else 16)
        run(p, 3 * d)
        for r in range(3):
            per, host = run(p)
            print(f"depth {d} streams {c} [{mode}]: {per:.4f} ms per evaluate, host {host:.4f} ms per submit", flush=True)
