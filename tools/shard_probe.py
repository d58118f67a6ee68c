"""Per-rank cost of the sharded evaluate at world sizes 1..8, emulated on ONE
GPU: each logical rank's PHASE_UP + PHASE_DOWN (its row strip of config 2) is
captured in a CUDA graph and replayed alone (L2 flushed in between), the
multipole / occupancy all-reduce replaced by nothing (its cost is NCCL's, not
measured here).  max over ranks ~ the per-step device time a W-GPU run would
see without the collective.  Usage: shard_probe.py [config] [worlds...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0809_1810_b200 as vf  # noqa: E402
from paper_0809_1810_b200 import distributed as D, workloads as W  # noqa: E402

cfg_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
worlds = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
w = W.by_index(cfg_idx)
dev = torch.device("cuda", 0)
cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
dom = vf.Domain(*W.DOMAIN)
x, y, g, s = (torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.Stream(dev)
for world in worlds:
    shards = D.make_shards(x, y, g, s, dom, cfg.levels, world)
    times = []
    for sh in shards:
        be = D.CudaShardBackend(dev, private_workspace=True)
        with torch.cuda.stream(stream):
            for _ in range(2):
                be.up(sh, cfg, dom)
                be.down(sh, cfg, dom, counters=False)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            be.up(sh, cfg, dom)
            be.down(sh, cfg, dom, counters=False)
        ts = []
        for _ in range(12):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            graph.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        times.append(statistics.median(ts[2:]))
    mx = max(times)
    print(f"{w.name} world {world}: per-rank ms min {min(times):.4f} max {mx:.4f} "
          f"-> {w.n / (mx * 1e-3) / 1e9:.2f} G evals/s without the all-reduce "
          f"(ranks: {' '.join(f'{t:.3f}' for t in times)})")

# phase times of the slowest rank of the largest world (stats mode, serialised)
if os.environ.get("PHASES"):
    import ctypes
    from paper_0809_1810_b200 import _lib
    from paper_0809_1810_b200._device import stream_ptr
    world = worlds[-1]
    shards = D.make_shards(x, y, g, s, dom, cfg.levels, world)
    lib = _lib.load()
    for r in (0, world // 2, world - 1):
        sh = shards[r]
        be = D.CudaShardBackend(dev, private_workspace=True)
        be.up(sh, cfg, dom)
        be.down(sh, cfg, dom, counters=False)
        torch.cuda.synchronize()
        vel = torch.zeros((2, sh.cols.shape[1]), dtype=torch.float64, device=dev)
        for ph, name in ((_lib.FLAG_PHASE_UP, "up"), (_lib.FLAG_PHASE_DOWN, "down")):
            st = _lib.VfmmStats()
            rc = lib.vfmm_evaluate_shard(*be._args(sh, cfg, dom), vel[0].data_ptr(), vel[1].data_ptr(),
                                         be.ws.ptr, be.ws.nbytes,
                                         ph | _lib.FLAG_STATS | _lib.FLAG_PHASE_TIMES, ctypes.byref(st),
                                         stream_ptr(dev))
            _lib.check(rc, "shard")
            print(f"world {world} rank {r} {name}: n_local {sh.cols.shape[1]} build {st.t_build*1e3:.4f} "
                  f"upward {st.t_upward*1e3:.4f} m2l {st.t_m2l*1e3:.4f} downward {st.t_downward*1e3:.4f} "
                  f"near {st.t_near*1e3:.4f} eval {st.t_eval*1e3:.4f} total {st.t_total*1e3:.4f}")
