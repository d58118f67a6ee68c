"""HostPipeline throughput (the bench's e2e) with the variants of the sigma
handling, plus the per-submit host cost.  Usage: pipe_e2e_probe.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import engine as E, workloads as W  # noqa: E402

w = W.by_index(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
dev = torch.device("cuda", 0)
n = w.n
dom = vf.Domain(*W.DOMAIN)
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
hx, hy, hg, hs = (torch.from_numpy(a).pin_memory() for a in (w.x, w.y, w.gamma, w.sigma))
t0 = time.perf_counter()
for _ in range(20):
    E._uniform_sigma((hs, hs.data_ptr()))
print(f"uniform-sigma host check: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per call")
for depth in (2, 3, 4):
    for scalar in (True, False):
        pipe = vf.HostPipeline(n, cfg, dom, depth=depth, device=dev)
        orig = E.evaluate_host_async

        def sub(x, y, g, s, _scalar=scalar):
            i = pipe.k % len(pipe.slots)
            pipe.k += 1
            if pipe.pending[i] is not None:
                pipe.pending[i].stream.synchronize()
            ws, stream, out = pipe.slots[i]
            pipe.pending[i] = orig(x, y, g, s, cfg, dom, out=out, workspace=ws, stream=stream,
                                   scalar_sigma=_scalar)
            return pipe.pending[i]

        for _ in range(2 * depth):
            sub(hx, hy, hg, hs)
        for p in pipe.pending:
            p.result()
        torch.cuda.synchronize()
        k = 30
        t0 = time.perf_counter()
        enq = 0.0
        for _ in range(k):
            a = time.perf_counter()
            sub(hx, hy, hg, hs)
            enq += time.perf_counter() - a
        for p in pipe.pending:
            p.result()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / k
        print(f"depth {depth} scalar_sigma {scalar}: {ms:.3f} ms per evaluate ({n / ms / 1e6:.3f} G/s), "
              f"host time in submit {enq / k * 1e3:.3f} ms")
