#!/usr/bin/env python
"""Benchmark: FMM particle velocity evaluations per second (fp64) on B200.

Workload (BASELINE.json configs[2], the configuration the metric is quoted on
at 1/2/4/8 B200): N = 1,048,576 particles on a 1024 x 1024 lattice over
[-1, 1]^2, two opposite-sign Lamb-Oseen vortices, sigma = h/0.8, l = 7,
p = 17, GAUSSIAN kernel, synthetic seeded inputs.

A step is one full ``evaluate`` (tree build, P2M, M2M, M2L, L2L, P2P, L2P,
combine) over the resident particle set.  ``value`` = N / mean step time with
inputs resident in HBM (CUDA graph replay of the C-ABI call; L2 flushed
between steps by writing a 256 MiB buffer outside the timed events).
``e2e`` = the same metric through the public host-buffer API
(``evaluate_host_async`` -> ``vfmm_evaluate_host``) with pinned HOST buffers:
every step copies x, y, gamma, sigma in (sigma as one value when all core
sizes are equal) and (u, v) out inside the timed region; eight independent
evaluations are kept in flight (``HostPipeline``: input copies on one H2D
stream, the evaluations' graphs on four compute streams, results on one D2H
stream), so one step's copies overlap its neighbours' compute.  ``e2e.latency_ms`` is one
synchronous ``evaluate_host`` call.

``--impl reference`` times the reference's CPU implementation on the SAME
workload: the unmodified ``vortexfmm`` package from its offline install under
baseline/_ref/ when present (it travels with the snapshot), else the numpy
oracle port in oracle/; one full config-2 evaluate per worker process per
step, one worker per host core.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "FMM particle velocity evals/sec (fp64)"
UNIT = "particle-evals/s"
P2P_FLOP_PER_PAIR_GAUSS = 42  # 14 basic + divide (8) + exp (20)
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: 64 DFMA/clk/SM at max clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2, choices=[0, 1, 2, 3])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-workers", type=int, default=0, help="reference arm: worker processes (0 = auto)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-depth", type=int, default=8, help="evaluations in flight in the e2e pipeline")
    ap.add_argument("--e2e-compute-streams", type=int, default=4,
                    help="compute streams of the e2e pipeline (0: one stream per slot for copies and compute)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU sharded path even for one rank (path check)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(idx):
    from paper_0809_1810_b200 import workloads as W

    return W.by_index(idx)


def host_info():
    """nproc, CPU model and memory of the host the CPU arms run on."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem_gb = None
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable"):
                    mem_gb = int(line.split()[1]) / 2**20
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return {"nproc": cores, "cpu_model": model, "mem_available_gb": mem_gb,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset")}


def time_oracle(w, repeats=1, blas_threads=1):
    """t_total of the numpy oracle port (the reference algorithm restated,
    oracle/fmm_oracle.py) on this host; ``blas_threads=None`` leaves the BLAS
    pool at its default (all cores), as the reference runs when
    OPENBLAS_NUM_THREADS is unset."""
    from threadpoolctl import threadpool_limits

    from oracle import fmm_oracle as O

    with threadpool_limits(limits=blas_threads):
        times = []
        for _ in range(repeats):
            _, st = O.evaluate(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, (-1.0, -1.0, 2.0))
            times.append(st["t_total"])
    return times


# ----------------------------------------------------------------- reference arm
_REF_W = None
_REF_LIMIT = None
REF_RSS_GB = {0: 0.3, 1: 0.5, 2: 1.5, 3: 24.0}  # measured peak RSS of one port evaluate (+ margin)


def _ref_package():
    """The UNMODIFIED reference package when its one offline install is present
    (tools/install_reference.sh -> git-ignored baseline/_ref/, which travels to
    the GPU box with the snapshot), else None (the numpy oracle port stands in)."""
    path = os.path.join(REPO, "baseline", "_ref")
    if os.environ.get("VFMM_REF_ARM") == "port" or not os.path.isdir(os.path.join(path, "vortexfmm")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import vortexfmm.engine as eng
        import vortexfmm.model as mod
    except Exception:  # a broken install: fall back to the port, and say so in `kind`
        return None
    return eng, mod


_REF_CALL = None


def _ref_init():
    """Per worker: one BLAS thread; with the reference installed, the particle
    list its public API takes (built once, outside the timed steps: it is the
    caller's input, not part of evaluate)."""
    global _REF_LIMIT, _REF_CALL
    from threadpoolctl import threadpool_limits

    _REF_LIMIT = threadpool_limits(limits=1)  # one BLAS thread per worker process
    w = _REF_W
    pkg = _ref_package()
    if pkg is not None:
        eng, mod = pkg
        ps = [mod.Particle(*t) for t in zip(w.x.tolist(), w.y.tolist(), w.gamma.tolist(), w.sigma.tolist())]
        cfg = eng.FmmConfig(w.levels, w.order, eng.KernelKind.GAUSSIAN_BLOB)
        dom = mod.Domain(-1.0, -1.0, 2.0)
        _REF_CALL = lambda: eng.evaluate(ps, cfg, dom)  # noqa: E731
    else:
        from oracle import fmm_oracle as O

        _REF_CALL = lambda: O.evaluate(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True,  # noqa: E731
                                       (-1.0, -1.0, 2.0))


def _ref_step(_):
    t0 = time.perf_counter()
    _REF_CALL()
    return time.perf_counter() - t0


def run_reference(args):
    """The reference's own CPU path on ALL host cores, on exactly our arm's
    workload.  With the reference's offline install present (baseline/_ref/,
    written by tools/install_reference.sh; `kind` = "reference") every worker
    calls the UNMODIFIED ``vortexfmm.engine.evaluate(list[Particle], FmmConfig,
    Domain)``; without it (`kind` = "port") the numpy oracle port runs instead
    (oracle/fmm_oracle.py, pinned to the reference at 1e-12 on the full config 2
    by tests/test_large_parity.py; ~1.7x faster than the reference itself).
    One worker process per core, one BLAS thread each: the reference is
    single-threaded apart from zgemm threads, which slow it down.
    A step is one FULL evaluate of the configuration per worker (N = 1,048,576,
    l = 7, p = 17 for config 2); value = workers x N / step wall time."""
    import multiprocessing as mp

    global _REF_W
    rank, world, _ = dist_env()
    if rank != 0:
        return
    _REF_W = w = workload(args.config)
    host = host_info()
    workers = max(1, min(host["nproc"], 64))
    if host["mem_available_gb"]:
        workers = max(1, min(workers, int(0.6 * host["mem_available_gb"] / REF_RSS_GB[args.config])))
    if args.ref_workers:
        workers = args.ref_workers
    t = []
    with mp.get_context("fork").Pool(workers, initializer=_ref_init) as pool:
        for _ in range(args.warmup):
            pool.map(_ref_step, range(workers))
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_ref_step, range(workers))
            t.append(time.perf_counter() - t0)
    mean = statistics.fmean(t)
    value = workers * w.n / mean
    kind = "reference" if _ref_package() is not None else "port"
    what = ("the unmodified vortexfmm.engine.evaluate (baseline/_ref)" if kind == "reference"
            else "the numpy oracle port")
    sample = (f"one full {w.name} evaluate (N={w.n}, l={w.levels}, p={w.order}) by {what} per worker per step, "
              f"{workers} worker processes x 1 BLAS thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": w.name, "n": w.n, "levels": w.levels, "order": w.order, "kernel": "gaussian",
                   "domain": [-1.0, -1.0, 2.0], "same_config": True},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": kind, "sample": sample,
                         "host": host},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- our arm
def fp64_peak(lib, torch, dev):
    """Measured DFMA throughput (TFLOP/s) of a dependent-chain probe filling all SMs."""
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flops = ctypes.c_double()
    blocks, iters = 148 * 8, 4096
    for _ in range(2):
        lib.vfmm_fp64_probe(sink.data_ptr(), blocks, iters, ctypes.byref(flops), stream.cuda_stream)
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(5):
        a.record(stream)
        lib.vfmm_fp64_probe(sink.data_ptr(), blocks, iters, ctypes.byref(flops), stream.cuda_stream)
        b.record(stream)
        b.synchronize()
        best = max(best, flops.value / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def run_ours(args):
    import torch

    import paper_0809_1810_b200 as vf
    from paper_0809_1810_b200 import _lib
    from paper_0809_1810_b200.engine import Workspace

    rank, world, local = dist_env()
    if world > 1 or args.sharded:
        from paper_0809_1810_b200 import distributed

        args.clock_sampler = ClockSampler  # clocks sampled on each rank's GPU in the timed region
        args.fp64_peak = fp64_peak          # roofline denominator, measured live per rank
        return distributed.bench_main(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _lib.load()
    w = workload(args.config)
    n = w.n
    cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
    dom = vf.Domain(-1.0, -1.0, 2.0)
    xd, yd, gd, sd = (torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
    out = torch.empty((2, n), dtype=torch.float64, device=dev)

    # warm-up with stats: counts, and the live per-phase CUDA-event times
    _, st = vf.evaluate_arrays(xd, yd, gd, sd, cfg, dom, out=out, timings=True)
    ws = Workspace.get(n, w.levels, w.order, dev)
    phase = []
    for _ in range(5):
        _, s = vf.evaluate_arrays(xd, yd, gd, sd, cfg, dom, out=out, timings=True)
        phase.append(s)
    t_near = statistics.fmean(p.t_near for p in phase)
    t_m2l = statistics.fmean(p.t_m2l for p in phase)

    # kernel launches per evaluate (host-side counter of the library)
    c0 = lib.vfmm_launch_count()
    stream = torch.cuda.Stream(dev)
    flags = _lib.FLAG_OVERLAP

    vel = torch.empty((n, 2), dtype=torch.float64, device=dev)  # (u, v) rows, the reference layout
    flags |= _lib.FLAG_UV_PAIRS

    def call(s):
        rc = lib.vfmm_evaluate(xd.data_ptr(), yd.data_ptr(), gd.data_ptr(), sd.data_ptr(), n,
                               dom.xmin, dom.ymin, dom.side, w.levels, w.order, _lib.KERNEL_GAUSSIAN,
                               vel.data_ptr(), None, ws.ptr, ws.nbytes, flags, None, s.cuda_stream)
        assert rc == 0, rc

    with torch.cuda.stream(stream):
        call(stream)
    torch.cuda.synchronize(dev)
    launches_per_step = lib.vfmm_launch_count() - c0

    graph = torch.cuda.CUDAGraph()
    c1 = lib.vfmm_launch_count()
    with torch.cuda.graph(graph, stream=stream):
        call(torch.cuda.current_stream(dev))
    # kernels a replay launches (the untaken paths sit in conditional nodes)
    graph_launches = lib.vfmm_launch_count() - c1
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(max(3, args.warmup)):
        flush.zero_()
        graph.replay()
    torch.cuda.synchronize(dev)
    ref_vel = vel.clone()
    assert torch.equal(vel.t(), out), "pair layout differs from the (2, N) layout"

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    cur = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for a, b in ev:
            flush.zero_()
            a.record(cur)
            graph.replay()
            b.record(cur)
        torch.cuda.synchronize(dev)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = statistics.fmean(step_ms)
    assert torch.equal(vel, ref_vel), "graph replays are not bitwise reproducible"

    # the phases as the graph runs them: the same call captured with its phase
    # events as event-record nodes (VFMM_FLAG_GRAPH_PHASES), replayed alone
    # (L2 flushed); elapsed from the call's start to each phase's end
    gflags = flags | _lib.FLAG_GRAPH_PHASES
    pgraph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(pgraph, stream=stream):
        rc = lib.vfmm_evaluate(xd.data_ptr(), yd.data_ptr(), gd.data_ptr(), sd.data_ptr(), n,
                               dom.xmin, dom.ymin, dom.side, w.levels, w.order, _lib.KERNEL_GAUSSIAN,
                               vel.data_ptr(), None, ws.ptr, ws.nbytes, gflags, None,
                               torch.cuda.current_stream(dev).cuda_stream)
        assert rc == 0, rc
    gph = []
    for _ in range(7):
        flush.zero_()
        pgraph.replay()
        torch.cuda.synchronize(dev)
        buf = (ctypes.c_float * 8)()
        assert lib.vfmm_graph_phase_times(local, buf) == 0
        gph.append(list(buf))
    gph = gph[2:]
    names = ("built", "upward", "m2l", "downward", "near_joined", "end", "near_start", "near_end")
    graph_phases = {k: statistics.fmean(r[i] for r in gph) for i, k in enumerate(names)}
    del pgraph

    # throughput of INDEPENDENT resident evaluations sharing the GPU (what the e2e
    # pipeline's compute stage does): four input sets (4 x 32 B x N > L2, so no step finds
    # its inputs in L2) with their own workspace and graph, replayed round robin on three
    # streams; the latency-bound head and tail of one evaluate hide behind the near field
    # of its neighbours.  Reported beside `value` (which stays one evaluate at a time).
    ov = []
    for _ in range(4):
        ins = [t.clone() for t in (xd, yd, gd, sd)]
        wsk = Workspace(n, w.levels, w.order, dev)
        velk = torch.empty((n, 2), dtype=torch.float64, device=dev)
        gk = torch.cuda.CUDAGraph()
        sk = torch.cuda.Stream(dev)

        def callk(s_, ins=ins, wsk=wsk, velk=velk):
            rc_ = lib.vfmm_evaluate(ins[0].data_ptr(), ins[1].data_ptr(), ins[2].data_ptr(), ins[3].data_ptr(),
                                    n, dom.xmin, dom.ymin, dom.side, w.levels, w.order, _lib.KERNEL_GAUSSIAN,
                                    velk.data_ptr(), None, wsk.ptr, wsk.nbytes, flags, None, s_.cuda_stream)
            assert rc_ == 0, rc_

        with torch.cuda.stream(sk):
            callk(sk)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(gk, stream=sk):
            callk(torch.cuda.current_stream(dev))
        ov.append((gk, velk, ins, wsk))
    ov_streams = [torch.cuda.Stream(dev) for _ in range(3)]

    def ov_run(k_steps):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a_.record(cur)
        for s_ in ov_streams:
            s_.wait_stream(cur)
        for k in range(k_steps):
            with torch.cuda.stream(ov_streams[k % 3]):
                ov[k % 4][0].replay()
        for s_ in ov_streams:
            cur.wait_stream(s_)
        b_.record(cur)
        b_.synchronize()
        return a_.elapsed_time(b_) / k_steps

    ov_run(8)
    ov_steps = max(12, args.steps)
    ov_ms = ov_run(ov_steps)
    for _, velk, _, _ in ov:
        assert torch.equal(velk, ref_vel), "overlapped replays differ"
    del ov

    # end to end through the public API from pinned host buffers
    hx, hy, hg, hs = (torch.from_numpy(a).pin_memory() for a in (w.x, w.y, w.gamma, w.sigma))
    host_out = torch.empty((n, 2), dtype=torch.float64).pin_memory()
    e2e_ms = []
    for i in range(args.e2e_steps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        vf.evaluate_host(hx, hy, hg, hs, cfg, dom, out=host_out, overlap=True)
        b.record(cur)
        b.synchronize()
        if i >= 2:
            e2e_ms.append(a.elapsed_time(b))
    assert torch.equal(host_out, ref_vel.cpu())
    e2e_latency = statistics.fmean(e2e_ms)
    # the reference's own signature: evaluate(list[Particle], FmmConfig, Domain)
    # -> (numpy (N, 2), FmmRunStats), list -> arrays conversion and the numpy
    # result included (SURVEY.md §8d asks for it beside the array paths)
    parts = [vf.Particle(float(a), float(b), float(c), float(d))
             for a, b, c, d in zip(w.x, w.y, w.gamma, w.sigma)]
    sig_ms = []
    for i in range(3):
        t0 = time.perf_counter()
        vnp, _ = vf.evaluate(parts, cfg, dom)
        sig_ms.append((time.perf_counter() - t0) * 1e3)
    assert np.array_equal(vnp, ref_vel.cpu().numpy()) or np.abs(vnp - ref_vel.cpu().numpy()).max() <= 1e-12 * np.abs(vnp).max()
    sig_ms = statistics.fmean(sig_ms[1:])
    del parts
    # throughput of a batch of independent evaluations through the async API:
    # HostPipeline keeps --e2e-depth calls in flight (own workspace, stream, pinned
    # output), so step k's H2D / D2H overlap the compute of its neighbours;
    # every step still copies its four input arrays in and its (N, 2) result out
    pipe = vf.HostPipeline(n, cfg, dom, depth=args.e2e_depth, device=dev,
                           compute_streams=args.e2e_compute_streams)
    k_pipe = max(8 * args.e2e_depth, args.e2e_steps)
    # untimed: every slot's first call (stream launches), its graph capture (second call)
    # and one replay
    for _ in range(3 * args.e2e_depth):
        pipe.submit(hx, hy, hg, hs)
    for p in pipe.pending:
        p.result()
    torch.cuda.synchronize(dev)
    # three batches of k_pipe steps, each timed on its own; the median is reported
    # (and all three kept in the line): PCIe-bound, a batch now and then reads ~7%
    # slower on this pool's hosts
    e2e_batches = []
    for _ in range(3):
        t0 = time.perf_counter()
        pend = [pipe.submit(hx, hy, hg, hs) for _ in range(k_pipe)]
        for p in pipe.pending:
            p.result()
        torch.cuda.synchronize(dev)
        e2e_batches.append((time.perf_counter() - t0) * 1e3 / k_pipe)
    e2e = statistics.median(e2e_batches)
    assert torch.equal(pend[-1].out, ref_vel.cpu()), "pipelined result differs"
    # a uniform sigma array travels as one value (VFMM_FLAG_SIGMA_SCALAR)
    sigma_uniform = bool((w.sigma.view(np.int64) == w.sigma.view(np.int64)[0]).all())

    peak = fp64_peak(lib, torch, dev)
    achieved = P2P_FLOP_PER_PAIR_GAUSS * st.near_pair_count / t_near / 1e12  # t_near in s
    # traffic and the executed FP64-pipe fraction of the dominant kernel: from
    # the committed `ncu --set full` capture of the same kernel and config
    # (profiles/p2p_traffic_config<c>.json, written by tools/ncu_summary.py);
    # a bench run cannot profile itself
    traffic = None
    ncu = {}
    prof = os.path.join(REPO, "profiles", f"p2p_traffic_config{args.config}.json")
    if os.path.exists(prof):
        try:
            ncu = json.load(open(prof))
            traffic = ncu.get("dram_bytes_per_launch")
        except Exception:
            traffic, ncu = None, {}
    m2l_flops = 8 * (w.order + 1) ** 2 * st.m2l_count
    hbm = None
    try:
        hbm = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        hbm = 6457.7  # this pool's measured copy bandwidth (round 1 MEASURED_PEAKS.json)
    # the build as it runs in the graph replay (untaken sort path not launched);
    # the stats-mode stream launch also runs the idle LSD kernels
    t_build = graph_phases["built"] * 1e-3 if graph_phases["built"] > 0 else \
        statistics.fmean(p.t_build for p in phase)
    build_bytes = 80 * n  # read x, y, Gamma, sigma; write the sorted copy; perm / keys
    # whole-pipeline roofline: FP64 work at the FP64 peak + the tree build's bytes at HBM
    # (T_roof = sum(FP64 flops) / F64_peak + tree_bytes / HBM)
    fp64_flops = (P2P_FLOP_PER_PAIR_GAUSS * st.near_pair_count + m2l_flops
                  + (8 * w.order + 4) * n + (8 * w.order + 6) * n
                  + 2 * 4 * (w.order + 1) * (w.order + 2) * sum(4**k for k in range(3, w.levels + 1)))
    t_roof = fp64_flops / (peak * 1e12) + build_bytes / (hbm * 1e9)

    cpu = None
    if not args.no_cpu_baseline:
        tt = time_oracle(w)[0]
        t_all = time_oracle(w, blas_threads=None)[0]
        cpu = {"value": n / tt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"one full {w.name} evaluate (N={n}) by the numpy oracle port, 1 BLAS thread",
               "blas_default_value": n / t_all, "host": host_info()}
        pkg = _ref_package()
        if pkg is not None:
            # the unmodified reference itself when its offline install travelled with the repo
            # (baseline/_ref): one full evaluate through its public API, 1 BLAS thread
            from threadpoolctl import threadpool_limits

            eng, mod = pkg
            ps = [mod.Particle(*t) for t in zip(w.x.tolist(), w.y.tolist(), w.gamma.tolist(), w.sigma.tolist())]
            rcfg = eng.FmmConfig(w.levels, w.order, eng.KernelKind.GAUSSIAN_BLOB)
            with threadpool_limits(limits=1):
                t0 = time.perf_counter()
                rvel, _ = eng.evaluate(ps, rcfg, mod.Domain(-1.0, -1.0, 2.0))
                t_ref = time.perf_counter() - t0
            del ps
            rerr = float(np.abs(rvel - ref_vel.cpu().numpy()).max() / np.abs(rvel).max())
            cpu.update({"port_value": cpu["value"], "value": n / t_ref, "kind": "reference",
                        "sample": f"one full {w.name} evaluate (N={n}) by the unmodified "
                                  "vortexfmm.engine.evaluate (baseline/_ref), 1 BLAS thread",
                        "max_rel_diff_vs_gpu": rerr})

    line = {
        "metric": METRIC, "value": n / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n": n, "levels": w.levels, "order": w.order, "kernel": "gaussian",
                   "domain": [-1.0, -1.0, 2.0], "l2": "flushed between steps (256 MiB write)",
                   "graph": "CUDA graph replay, near field overlapped with far-field chain",
                   "m2l_count": st.m2l_count, "near_pair_count": st.near_pair_count},
        "e2e": {"value": n / (e2e * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": 3 * 8 * n + (8 if sigma_uniform else 8 * n),
                "d2h_bytes_per_step": 2 * 8 * n, "ms_per_step": e2e, "batches_ms_per_step": e2e_batches,
                "mode": f"evaluate_host_async via HostPipeline(depth={args.e2e_depth}, compute_streams="
                        f"{args.e2e_compute_streams}: input copies on one H2D stream, cached CUDA graph per slot "
                        f"on the compute streams, results on one D2H stream), median of 3 batches of {k_pipe} steps, host wall clock",
                "latency_ms": e2e_latency,
                "latency_mode": "one synchronous evaluate_host call (stats on; copies overlapped with the build), CUDA events",
                "reference_signature_ms": sig_ms,
                "reference_signature_mode": "evaluate(list[Particle], FmmConfig, Domain) -> (numpy (N, 2), stats): "
                                            "list -> arrays conversion, copies, evaluate, numpy result; host wall clock"},
        "overlapped": {"value": n / (ov_ms * 1e-3), "unit": UNIT, "ms_per_step": ov_ms, "steps": ov_steps,
                       "mode": "independent resident evaluates (4 input sets > L2, own workspace and CUDA graph) "
                               "replayed round robin on 3 streams; CUDA events around the batch"},
        "gpu_launches": int(graph_launches) * args.steps,
        "launches_per_step": {"graph_replay": int(graph_launches), "stream_call": int(launches_per_step)},
        "roofline": {"bound": "fp64", "kernel": "k_p2p (near field)", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "peak_source": "measured live: DFMA probe (vfmm_fp64_probe), 148x8 CTAs",
                     "nominal_peak": NOMINAL_FP64_TFLOPS,
                     "traffic": traffic, "p2p_ms": t_near * 1e3,
                     "flop_per_pair": P2P_FLOP_PER_PAIR_GAUSS,
                     "fp64_pipe_executed_pct": ncu.get("fp64_pipe_active_pct"),
                     "ncu_source": ncu.get("source"),
                     "m2l": {"achieved": m2l_flops / t_m2l / 1e12, "ms": t_m2l * 1e3,
                             "frac": m2l_flops / t_m2l / 1e12 / peak,
                             "flop_per_translation": 8 * (w.order + 1) ** 2},
                     "build": {"bound": "hbm", "achieved": build_bytes / t_build / 1e9, "ms": t_build * 1e3,
                               "peak": hbm, "unit": "GB/s", "frac": build_bytes / t_build / 1e9 / hbm,
                               "bytes_per_particle": 80,
                               "timed": "in the CUDA graph replay (event-record nodes, VFMM_FLAG_GRAPH_PHASES)"},
                     "step": {"t_roof_ms": t_roof * 1e3, "frac": t_roof / (ms * 1e-3),
                              "note": "sum of FP64 work at the live FP64 peak + build bytes at measured HBM, "
                                      "over the measured step"}},
        "phases_ms": {k: statistics.fmean(getattr(p, k) for p in phase) * 1e3 for k in
                      ("t_build", "t_upward", "t_m2l", "t_downward", "t_eval", "t_near", "t_total")},
        "phases_mode": "stats-mode stream launches, phases serialised by events (idle LSD kernels included)",
        "graph_timeline_ms": graph_phases,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
