"""Graph replay of one evaluate with / without per-node priorities (timing experiment)."""
import os
import sys
import statistics

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import _lib, workloads as W  # noqa: E402
from paper_0809_1810_b200.engine import Workspace  # noqa: E402

w = W.by_index(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
dev = torch.device("cuda", 0)
xd, yd, gd, sd = (torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
n = xd.numel()
lib = _lib.load()
ws = Workspace.get(n, w.levels, w.order, dev)
dom = vf.Domain(*W.DOMAIN)
vel = torch.empty((n, 2), dtype=torch.float64, device=dev)
stream = torch.cuda.Stream(dev)
flags = _lib.FLAG_OVERLAP | _lib.FLAG_UV_PAIRS


def call(s):
    rc = lib.vfmm_evaluate(xd.data_ptr(), yd.data_ptr(), gd.data_ptr(), sd.data_ptr(), n, dom.xmin,
                           dom.ymin, dom.side, w.levels, w.order, _lib.KERNEL_GAUSSIAN, vel.data_ptr(),
                           None, ws.ptr, ws.nbytes, flags, None, s)
    assert rc == 0, rc


with torch.cuda.stream(stream):
    call(stream.cuda_stream)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for use_prio in (False, True, False, True):
    err, = rt.cudaStreamBeginCapture(stream.cuda_stream, rt.cudaStreamCaptureMode.cudaStreamCaptureModeGlobal)[:1]
    call(stream.cuda_stream)
    err, graph = rt.cudaStreamEndCapture(stream.cuda_stream)
    fl = rt.cudaGraphInstantiateFlags.cudaGraphInstantiateFlagUseNodePriority if use_prio else 0
    err, gexec = rt.cudaGraphInstantiateWithFlags(graph, int(fl))
    assert int(err) == 0, err
    times = []
    for i in range(25):
        with torch.cuda.stream(stream):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            rt.cudaGraphLaunch(gexec, stream.cuda_stream)
            b.record(stream)
        b.synchronize()
        if i >= 5:
            times.append(a.elapsed_time(b))
    print(f"node priorities {use_prio}: {statistics.fmean(times):.4f} ms")
    rt.cudaGraphExecDestroy(gexec)
    rt.cudaGraphDestroy(graph)
