"""Three-stage host pipeline experiment: H2D on a copy stream, the captured
evaluate on C compute streams (at most C evaluations share the SMs), D2H on a
second copy stream; D slots of buffers.  Per-step wall time for several (D, C).
Usage: pipe3_probe.py [config] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import _lib, workloads as W  # noqa: E402
from paper_0809_1810_b200.engine import Workspace  # noqa: E402

w = W.by_index(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 48
dev = torch.device("cuda", 0)
n = w.n
lib = _lib.load()
dom = vf.Domain(*W.DOMAIN)
flags = _lib.FLAG_OVERLAP | _lib.FLAG_UV_PAIRS
hx, hy, hg, hs = (torch.from_numpy(a).pin_memory() for a in (w.x, w.y, w.gamma, w.sigma))
MAXD = 8


class Slot:
    def __init__(self):
        self.ws = Workspace(n, w.levels, w.order, dev)
        self.din = torch.empty((4, n), dtype=torch.float64, device=dev)
        self.din[3].copy_(hs)
        self.vel = torch.empty((n, 2), dtype=torch.float64, device=dev)
        self.out = torch.empty((n, 2), dtype=torch.float64).pin_memory()
        self.in_ready, self.done, self.out_ready = (torch.cuda.Event() for _ in range(3))
        cap = torch.cuda.Stream(dev)
        self.call(cap.cuda_stream)
        torch.cuda.synchronize()
        rt.cudaStreamBeginCapture(cap.cuda_stream, rt.cudaStreamCaptureMode.cudaStreamCaptureModeGlobal)
        self.call(cap.cuda_stream)
        err, graph = rt.cudaStreamEndCapture(cap.cuda_stream)
        err, self.gexec = rt.cudaGraphInstantiateWithFlags(graph, 0)
        assert int(err) == 0, err

    def call(self, s):
        d = self.din
        rc = lib.vfmm_evaluate(d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), n, dom.xmin,
                               dom.ymin, dom.side, w.levels, w.order, _lib.KERNEL_GAUSSIAN,
                               self.vel.data_ptr(), None, self.ws.ptr, self.ws.nbytes, flags, None, s)
        assert rc == 0, rc


slots = [Slot() for _ in range(MAXD)]
for s in slots:
    s.din[:3].zero_()
h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
comp = [torch.cuda.Stream(dev) for _ in range(4)]
ref = None


def run(D, C, k_steps, sigma_too):
    for s in slots:
        s.out_ready.record(d2h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(k_steps):
        s = slots[k % D]
        s.out_ready.synchronize()  # the slot's previous result has left the device
        with torch.cuda.stream(h2d):
            s.din[0].copy_(hx, non_blocking=True)
            s.din[1].copy_(hy, non_blocking=True)
            s.din[2].copy_(hg, non_blocking=True)
            if sigma_too:
                s.din[3].copy_(hs, non_blocking=True)
            s.in_ready.record(h2d)
        cs = comp[k % C]
        cs.wait_event(s.in_ready)
        rt.cudaGraphLaunch(s.gexec, cs.cuda_stream)
        s.done.record(cs)
        d2h.wait_event(s.done)
        with torch.cuda.stream(d2h):
            s.out.copy_(s.vel, non_blocking=True)
            s.out_ready.record(d2h)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / k_steps


for sigma_too in (False, True):
    for D, C in ((2, 2), (3, 3), (4, 2), (4, 3), (4, 4), (6, 2), (6, 3), (8, 2), (8, 3), (8, 4)):
        run(D, C, 2 * D, sigma_too)
        per = run(D, C, steps, sigma_too)
        if ref is None:
            ref = slots[0].out.clone()
        print(f"slots {D} compute streams {C} sigma copied {sigma_too}: {per:.4f} ms per evaluate "
              f"({n / per / 1e6:.1f} M particle-evals/s)", flush=True)
for s in slots:
    assert torch.equal(s.out, ref), "results differ between slots"
print("all slots bitwise equal")
