"""One full evaluate of a BASELINE config (default 2) captured as a CUDA graph
(the bench's timed form: near field overlapped with the far chain, untaken
paths in conditional nodes) and replayed `reps` times -- for ncu launch lists
and --set full captures of the kernels as they run in the bench.
Usage: profile_graph.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import _lib, workloads as W  # noqa: E402
from paper_0809_1810_b200.engine import Workspace  # noqa: E402

cfg_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = W.by_index(cfg_idx)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
lib = _lib.load()
xd, yd, gd, sd = (torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
vf.evaluate_arrays(xd, yd, gd, sd, cfg, vf.Domain(*W.DOMAIN))  # tables, workspace
ws = Workspace.get(w.n, w.levels, w.order, dev)
vel = torch.empty((w.n, 2), dtype=torch.float64, device=dev)
stream = torch.cuda.Stream(dev)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=stream):
    rc = lib.vfmm_evaluate(xd.data_ptr(), yd.data_ptr(), gd.data_ptr(), sd.data_ptr(), w.n, -1.0, -1.0, 2.0,
                           w.levels, w.order, _lib.KERNEL_GAUSSIAN, vel.data_ptr(), None, ws.ptr, ws.nbytes,
                           _lib.FLAG_OVERLAP | _lib.FLAG_UV_PAIRS, None,
                           torch.cuda.current_stream(dev).cuda_stream)
    assert rc == 0, rc
for _ in range(reps):
    graph.replay()
torch.cuda.synchronize()
print(f"{w.name}: {reps} graph replays, |v|max = {float(vel.abs().max()):.6e}")
