"""HostPipeline throughput probe: per-step wall time, host time per submit."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0809_1810_b200 as vf
from paper_0809_1810_b200 import workloads as W, engine
w = W.by_index(2)
dev = torch.device("cuda", 0)
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
dom = vf.Domain(*W.DOMAIN)
hx, hy, hg, hs = (torch.from_numpy(a).pin_memory() for a in (w.x, w.y, w.gamma, w.sigma))
for depth in (2, 3, 4):
    for scalar in (False, True):
        pipe = vf.HostPipeline(w.n, cfg, dom, depth=depth, device=dev)
        def submit():
            i = pipe.k % len(pipe.slots)
            pipe.k += 1
            if pipe.pending[i] is not None:
                pipe.pending[i].result()
            ws, stream, out = pipe.slots[i]
            t = time.perf_counter()
            pipe.pending[i] = engine.evaluate_host_async(hx, hy, hg, hs, cfg, dom, out=out, workspace=ws,
                                                         stream=stream, scalar_sigma=scalar)
            return time.perf_counter() - t
        for _ in range(depth + 1):
            submit()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host = [submit() for _ in range(24)]
        for p in pipe.pending:
            p.result()
        torch.cuda.synchronize()
        per = (time.perf_counter() - t0) * 1e3 / 24
        print(f"depth {depth} scalar_sigma {scalar}: {per:.3f} ms/step, host submit {statistics.fmean(host)*1e3:.3f} ms")
