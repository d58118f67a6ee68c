"""vfmm_evaluate_host_streams called directly (no engine.py) in the three-stage
layout, with toggles, to separate the library's cost from the Python host path.
Usage: pipe_c_probe.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import _lib, workloads as W  # noqa: E402
from paper_0809_1810_b200.engine import Workspace  # noqa: E402

w = W.by_index(2)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda", 0)
n = w.n
lib = _lib.load()
dom = vf.Domain(*W.DOMAIN)
hx, hy, hg, hs = (torch.from_numpy(a).pin_memory() for a in (w.x, w.y, w.gamma, w.sigma))
one = torch.full((1,), float(w.sigma[0]), dtype=torch.float64).pin_memory()
MAXD = 8
slots = [(Workspace(n, w.levels, w.order, dev), torch.empty((n, 2), dtype=torch.float64).pin_memory(),
          torch.cuda.Event(), torch.zeros(1, dtype=torch.int32).pin_memory()) for _ in range(MAXD)]
h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
comp = [torch.cuda.Stream(dev) for _ in range(4)]


def run(D, C, k_steps, scalar, badcount):
    base = _lib.FLAG_OVERLAP | _lib.FLAG_UV_PAIRS | (_lib.FLAG_SIGMA_SCALAR if scalar else 0)
    sp = one.data_ptr() if scalar else hs.data_ptr()
    for s in slots:
        s[2].record(d2h)
    torch.cuda.synchronize()
    host = 0.0
    t0 = time.perf_counter()
    for k in range(k_steps):
        ws, out, ev, bad = slots[k % D]
        ev.synchronize()
        t1 = time.perf_counter()
        rc = lib.vfmm_evaluate_host_streams(hx.data_ptr(), hy.data_ptr(), hg.data_ptr(), sp, n, dom.xmin,
                                            dom.ymin, dom.side, w.levels, w.order, _lib.KERNEL_GAUSSIAN,
                                            out.data_ptr(), None, ws.ptr, ws.nbytes, base,
                                            comp[k % C].cuda_stream, h2d.cuda_stream, d2h.cuda_stream)
        assert rc == 0, rc
        if badcount:
            lib.vfmm_bad_count_async(n, w.levels, w.order, ws.ptr, bad.data_ptr(), d2h.cuda_stream)
        ev.record(d2h)
        host += time.perf_counter() - t1
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / k_steps, host * 1e3 / k_steps


for scalar, badcount in ((True, True), (True, False), (False, False)):
    for D, C in ((3, 3), (4, 4), (6, 3), (8, 4)):
        run(D, C, 3 * D, scalar, badcount)
        for r in range(3):
            per, host = run(D, C, steps, scalar, badcount)
            print(f"scalar {scalar} badcount {badcount} slots {D} streams {C}: {per:.4f} ms per evaluate, "
                  f"host {host:.4f} ms per submit", flush=True)
