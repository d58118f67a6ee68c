"""Per-rank cost of the sharded evaluate at world sizes 1..8, emulated on ONE
GPU: each logical rank's PHASE_UP, pack, modelled exchange, unpack and
PHASE_DOWN (its row strip of the config) is captured in a CUDA graph and
replayed alone (L2 flushed in between).  The NCCL exchange is MODELLED by a
device spin (torch.cuda._sleep) on the caller's stream between pack and
unpack, so the near field (started by PHASE_UP on its own stream) overlaps
it as in a real run: t = alpha_ag + world * coarse_bytes / B (allgather,
when there are coarse levels) + alpha_p2p + halo_bytes / B (neighbour send /
recv), B = 770 GB/s per direction (measured peer copy, B200_PROFILING.md),
alpha_ag = 12 us, alpha_p2p = 8 us (assumed NCCL small-message latencies).
The unpack reads the rank's own send buffers in place of its neighbours'
(same sizes).  max over ranks ~ the per-step device time of a W-GPU run.
Usage: shard_probe.py [config] [worlds...]"""
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
B = 770e9
ALPHA_AG, ALPHA_P2P = 12e-6, 8e-6
sm_hz = torch.cuda.get_device_properties(dev).clock_rate * 1e3  # kHz -> Hz
for world in worlds:
    shards = D.make_shards(x, y, g, s, dom, cfg.levels, world)
    bounds = D.row_bounds(cfg.levels, world)
    kc = D.coarse_cut(cfg.levels, bounds)
    times, xbytes = [], []
    for r, sh in enumerate(shards):
        be = D.CudaShardBackend(dev, private_workspace=True)
        below, above = D.neighbours(bounds, r)

        def step():
            be.up(sh, cfg, dom)
            coarse, down, up = be.pack(kc, below is not None, above is not None)
            t_x = 0.0
            if coarse is not None and world > 1:
                t_x += ALPHA_AG + world * coarse.numel() / B
            hb = sum(t.numel() for t in (down, up) if t is not None)
            if hb:
                t_x += ALPHA_P2P + hb / B
            if t_x > 0:
                torch.cuda._sleep(int(t_x * sm_hz))
            ca = torch.cat([coarse] * world) if coarse is not None else None
            be.unpack(kc, ca, world, up if below is not None else None,
                      down if above is not None else None)
            be.down(sh, cfg, dom, counters=False)
            return t_x, (0 if coarse is None else world * coarse.numel()) + hb

        with torch.cuda.stream(stream):
            for _ in range(2):
                t_x, nbytes = step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
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
        xbytes.append((nbytes, t_x))
    mx = max(times)
    mb = max(b for b, _ in xbytes) / 1e6
    print(f"{w.name} world {world} (kc {kc}): per-rank ms min {min(times):.4f} max {mx:.4f} "
          f"-> {w.n / (mx * 1e-3) / 1e9:.2f} G evals/s; exchange received per rank <= {mb:.3f} MB, "
          f"modelled {max(t for _, t in xbytes) * 1e6:.1f} us (ranks: {' '.join(f'{t:.3f}' for t in times)})")

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
