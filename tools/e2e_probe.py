"""Where the end-to-end (host buffers) time goes: enqueue cost, stats sync, copies."""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import _lib, workloads as W  # noqa: E402
from paper_0809_1810_b200.engine import Workspace  # noqa: E402
from paper_0809_1810_b200._device import stream_ptr  # noqa: E402

w = W.by_index(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
dev = torch.device("cuda", 0)
n = w.x.size
lib = _lib.load()
ws = Workspace.get(n, w.levels, w.order, dev)
dom = vf.Domain(*W.DOMAIN)
hx, hy, hg, hs = (torch.from_numpy(a).pin_memory() for a in (w.x, w.y, w.gamma, w.sigma))
out = torch.empty((n, 2), dtype=torch.float64).pin_memory()
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
s = stream_ptr(dev)


def raw(flags, st=None):
    return lib.vfmm_evaluate_host(hx.data_ptr(), hy.data_ptr(), hg.data_ptr(), hs.data_ptr(), n, dom.xmin,
                                  dom.ymin, dom.side, w.levels, w.order, _lib.KERNEL_GAUSSIAN,
                                  out.data_ptr(), None, ws.ptr, ws.nbytes, flags, st, s)


for name, flags, use_st in [("public evaluate_host", None, None),
                            ("raw, no stats", _lib.FLAG_OVERLAP | _lib.FLAG_UV_PAIRS, False),
                            ("raw, stats", _lib.FLAG_OVERLAP | _lib.FLAG_UV_PAIRS | _lib.FLAG_STATS, True)]:
    wall, enq = [], []
    for i in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if flags is None:
            vf.evaluate_host(hx, hy, hg, hs, cfg, dom, out=out, overlap=True)
        else:
            st = _lib.VfmmStats()
            rc = raw(flags, ctypes.byref(st) if use_st else None)
            assert rc == 0, rc
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if i >= 2:
            enq.append((t1 - t0) * 1e3)
            wall.append((t2 - t0) * 1e3)
    print(f"{name:24s} wall {statistics.fmean(wall):.3f} ms  (call returns after {statistics.fmean(enq):.3f} ms)")
# pure copies
a = torch.empty(4 * n, dtype=torch.float64, device=dev)
hb = torch.empty(4 * n, dtype=torch.float64).pin_memory()
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); a.copy_(hb, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); hb[: 2 * n].copy_(a[: 2 * n], non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"H2D {32 * n / 1e6:.0f} MB: {(t1 - t0) * 1e3:.3f} ms, D2H {16 * n / 1e6:.0f} MB: {(t2 - t1) * 1e3:.3f} ms")
_, st = vf.evaluate_host(hx, hy, hg, hs, cfg, dom, out=out, overlap=True)
print({k: round(v * 1e3, 4) for k, v in vars(st).items() if k.startswith("t_")})
