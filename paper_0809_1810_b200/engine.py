"""Drop-in FMM engine: ``evaluate`` / ``evaluate_at`` on the B200.

Mirrors ``vortexfmm.engine`` (reference ``engine.py:41-74,335-460``):
same ``FmmConfig`` / ``FmmRunStats`` fields, same argument validation and
error types (``ValueError``, ``OutOfDomainError``), the same sigma-guard
``UserWarning`` text, and the same return value -- an (N, 2) float64 array of
(u, v) in the caller's particle order plus the run statistics.

Every phase runs in the CUDA library (``libvfmm.so``, ``csrc/``) through the
C ABI of ``include/vfmm.h``; this module only converts inputs, owns the
device workspace and maps status codes to the reference's exceptions.
"""

from __future__ import annotations

import ctypes
import threading
import warnings
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from ._device import as_device_f64, device_of, require_cuda, stream_ptr, torch
from .kernels import KernelKind, kernel_code
from .model import Domain, enclosing_domain_of, to_arrays
from .quadtree import OutOfDomainError

ORDER_CAP = _lib.ORDER_CAP


@dataclass(frozen=True)
class FmmConfig:
    """Run parameters: tree depth, truncation order, near-field kernel (engine.py:41-55)."""

    levels: int
    order: int
    kernel: KernelKind = KernelKind.POINT_VORTEX

    def validate(self) -> None:
        validate_config(self)


def validate_config(config) -> None:
    """FmmConfig.validate (engine.py:49-55) for our or the reference's config."""
    if config.levels < 2:
        raise ValueError(f"levels must be >= 2, got {config.levels}")
    if config.order < 0:
        raise ValueError(f"order must be >= 0, got {config.order}")
    if config.order > ORDER_CAP:
        raise ValueError(f"order {config.order} exceeds cap {ORDER_CAP}")
    if config.levels > _lib.LEVELS_CAP:
        raise ValueError(f"levels {config.levels} exceeds the GPU tree cap {_lib.LEVELS_CAP}")
    kernel_code(config.kernel)


@dataclass
class FmmRunStats:
    """Phase timings (seconds, CUDA events) and exact counters (engine.py:58-74)."""

    n: int
    levels: int
    order: int
    t_build: float = 0.0
    t_upward: float = 0.0
    t_m2l: float = 0.0
    t_downward: float = 0.0
    t_eval: float = 0.0
    t_near: float = 0.0
    t_total: float = 0.0
    m2l_count: int = 0
    near_pair_count: int = 0
    sigma_guard_ok: bool = True


class Workspace:
    """Device scratch for one (n, levels, order) shape, reused across calls.

    The cache is keyed by host thread as well: a workspace holds the whole
    state of one evaluate, so two threads evaluating at once never share one
    (the library serialises their enqueue, include/vfmm.h "Threading")."""

    _cache: dict = {}
    _cache_lock = threading.Lock()

    def __init__(self, n: int, levels: int, order: int, device: torch.device):
        self.n, self.levels, self.order, self.device = n, levels, order, device
        self.nbytes = _lib.workspace_size(n, levels, order)
        self.buffer = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.layout = _lib.layout(n, levels, order)

    @property
    def ptr(self) -> int:
        return self.buffer.data_ptr()

    @classmethod
    def get(cls, n: int, levels: int, order: int, device: torch.device) -> "Workspace":
        key = (threading.get_ident(), device.index, n, levels, order)
        with cls._cache_lock:
            ws = cls._cache.get(key)
            if ws is None:
                if len(cls._cache) >= 4:
                    cls._cache.pop(next(iter(cls._cache)))
                ws = cls(n, levels, order, device)
                cls._cache[key] = ws
            return ws

    # ---- typed views of the internal arrays (parity tests / debugging) ----
    def view(self, name: str, dtype: torch.dtype, count: int) -> torch.Tensor:
        off = getattr(self.layout, name)
        esize = torch.empty(0, dtype=dtype).element_size()
        return self.buffer[off: off + count * esize].view(dtype)


def _bad_indices(x, y, domain) -> np.ndarray:
    x = x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
    y = y.cpu().numpy() if isinstance(y, torch.Tensor) else np.asarray(y)
    inside = (x >= domain.xmin) & (x <= domain.xmax) & (y >= domain.ymin) & (y <= domain.ymax)
    return np.flatnonzero(~inside)


def _stats_from(c: _lib.VfmmStats) -> FmmRunStats:
    return FmmRunStats(
        n=int(c.n),
        levels=int(c.levels),
        order=int(c.order),
        t_build=c.t_build * 1e-3,
        t_upward=c.t_upward * 1e-3,
        t_m2l=c.t_m2l * 1e-3,
        t_downward=c.t_downward * 1e-3,
        t_eval=c.t_eval * 1e-3,
        t_near=c.t_near * 1e-3,
        t_total=c.t_total * 1e-3,
        m2l_count=int(c.m2l_count),
        near_pair_count=int(c.near_pair_count),
        sigma_guard_ok=bool(c.sigma_guard_ok),
    )


def evaluate_arrays(
    x,
    y,
    gamma,
    sigma,
    config,
    domain=None,
    *,
    device=None,
    overlap: bool = False,
    out: torch.Tensor | None = None,
    timings: bool = False,
    stacklevel: int = 2,
):
    """Array fast path of :func:`evaluate`.

    ``x, y, gamma, sigma`` are length-N numpy arrays or torch tensors (CUDA
    tensors are used in place).  Returns ``(vel, stats)`` where ``vel`` is a
    (2, N) float64 CUDA tensor holding u (row 0) and v (row 1) in the input
    order.  ``overlap=True`` runs the near field concurrently with the
    far-field chain (phase timings then overlap in time).  ``timings=True``
    fills the per-phase times of ``stats`` (CUDA events between the phases,
    ~0.1 ms per call); otherwise only ``t_total`` and the counters.
    """
    validate_config(config)
    require_cuda()
    lib = _lib.load()
    dev = device_of(device, x)
    xd, yd, gd = (as_device_f64(a, dev) for a in (x, y, gamma))
    n = int(xd.numel())
    if n == 0:
        raise ValueError("need at least one particle")
    code = kernel_code(config.kernel)
    sd = as_device_f64(sigma, dev) if code == _lib.KERNEL_GAUSSIAN else None
    if domain is None:
        domain = enclosing_domain_of(xd.cpu().numpy(), yd.cpu().numpy())
    ws = Workspace.get(n, config.levels, config.order, dev)
    if out is None:
        out = torch.empty((2, n), dtype=torch.float64, device=dev)
    st = _lib.VfmmStats()
    flags = _lib.FLAG_STATS | (_lib.FLAG_OVERLAP if overlap else 0) | (_lib.FLAG_PHASE_TIMES if timings else 0)
    status = lib.vfmm_evaluate(
        xd.data_ptr(), yd.data_ptr(), gd.data_ptr(), sd.data_ptr() if sd is not None else None, n,
        float(domain.xmin), float(domain.ymin), float(domain.side), config.levels, config.order,
        code, out[0].data_ptr(), out[1].data_ptr(), ws.ptr, ws.nbytes, flags, ctypes.byref(st),
        stream_ptr(dev),
    )
    if status == _lib.VFMM_EDOMAIN:
        bad = _bad_indices(xd, yd, domain)
        raise OutOfDomainError(
            f"{bad.size} particle(s) outside domain {domain}, first indices {bad[:5].tolist()}"
        )
    _lib.check(status, "vfmm_evaluate")
    stats = _stats_from(st)
    if code == _lib.KERNEL_GAUSSIAN and not st.sigma_guard_ok:
        warnings.warn(
            f"max core radius {st.max_sigma:g} exceeds leaf half-width/2 = {st.sigma_guard:g}; "
            "the far field treats blobs as point vortices, so expect extra error",
            stacklevel=stacklevel + 1,
        )
    return out, stats


def _host_f64(a) -> tuple[object, int]:
    """(keep-alive object, data pointer) of a contiguous float64 host array."""
    if isinstance(a, torch.Tensor):
        t = a.detach().to(torch.float64).contiguous()
        if t.is_cuda:
            raise ValueError("evaluate_host takes host arrays; use evaluate_arrays for device data")
        return t, t.data_ptr()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return arr, arr.ctypes.data


def evaluate_host(
    x,
    y,
    gamma,
    sigma,
    config,
    domain=None,
    *,
    device=None,
    out: torch.Tensor | None = None,
    overlap: bool = True,
    timings: bool = False,
    graph: bool | None = None,
    stacklevel: int = 2,
):
    """Host-buffer fast path (``vfmm_evaluate_host``): numpy arrays or CPU (ideally
    pinned) tensors in, an (N, 2) float64 host tensor of (u, v) rows out (the
    reference's return layout, engine.py:394-398).

    The library stages the copies itself and overlaps them with the tree
    build (positions first; circulations and core sizes while the sort runs).
    With ``graph`` the device part is replayed from a CUDA graph cached per
    workspace / shape / domain from the second call of a shape on
    (VFMM_FLAG_GRAPH): no launch gaps, but the input copies then all precede
    the compute instead of overlapping the build.  Default (None): graphs
    for N < 2^18, where launch overhead dominates; stream launches above,
    where the PCIe copies do (measured config 2: 1.75 ms stream vs 1.98 ms
    graph per synchronous call).  ``timings=True`` uses stream launches.
    """
    validate_config(config)
    require_cuda()
    lib = _lib.load()
    dev = device_of(device)
    keep = [_host_f64(a) for a in (x, y, gamma, sigma)]
    n = int(np.asarray(keep[0][0]).size) if not isinstance(keep[0][0], torch.Tensor) else keep[0][0].numel()
    if n == 0:
        raise ValueError("need at least one particle")
    if domain is None:
        xs = keep[0][0].numpy() if isinstance(keep[0][0], torch.Tensor) else keep[0][0]
        ys = keep[1][0].numpy() if isinstance(keep[1][0], torch.Tensor) else keep[1][0]
        domain = enclosing_domain_of(xs, ys)
    code = kernel_code(config.kernel)
    ws = Workspace.get(n, config.levels, config.order, dev)
    if out is None:
        out = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
    if tuple(out.shape) != (n, 2) or not out.is_contiguous() or out.is_cuda:
        raise ValueError("out must be a contiguous host (N, 2) float64 tensor")
    if graph is None:
        graph = n < (1 << 18)
    st = _lib.VfmmStats()
    flags = (_lib.FLAG_STATS | _lib.FLAG_UV_PAIRS | (_lib.FLAG_OVERLAP if overlap else 0)
             | (_lib.FLAG_PHASE_TIMES if timings else 0)
             | (_lib.FLAG_GRAPH if graph and not timings else 0))
    status = lib.vfmm_evaluate_host(
        keep[0][1], keep[1][1], keep[2][1], keep[3][1] if code == _lib.KERNEL_GAUSSIAN else None, n,
        float(domain.xmin), float(domain.ymin), float(domain.side), config.levels, config.order,
        code, out.data_ptr(), None, ws.ptr, ws.nbytes, flags, ctypes.byref(st), stream_ptr(dev),
    )
    if status == _lib.VFMM_EDOMAIN:
        xs = keep[0][0].numpy() if isinstance(keep[0][0], torch.Tensor) else keep[0][0]
        ys = keep[1][0].numpy() if isinstance(keep[1][0], torch.Tensor) else keep[1][0]
        bad = _bad_indices(xs, ys, domain)
        raise OutOfDomainError(
            f"{bad.size} particle(s) outside domain {domain}, first indices {bad[:5].tolist()}"
        )
    _lib.check(status, "vfmm_evaluate_host")
    stats = _stats_from(st)
    if code == _lib.KERNEL_GAUSSIAN and not st.sigma_guard_ok:
        warnings.warn(
            f"max core radius {st.max_sigma:g} exceeds leaf half-width/2 = {st.sigma_guard:g}; "
            "the far field treats blobs as point vortices, so expect extra error",
            stacklevel=stacklevel + 1,
        )
    return out, stats


class PendingEvaluation:
    """An :func:`evaluate_host_async` call in flight; :meth:`result` waits for it."""

    def __init__(self, out, stream, keep, ws, config, domain, n, code, bad, event=None):
        self.out, self.stream, self._keep, self.ws = out, stream, keep, ws
        self._config, self._domain, self._n, self._code = config, domain, n, code
        self._bad = bad  # pinned int32: out-of-domain count, copied on the stream
        # three-stream calls: recorded on the D2H copy stream (shared by the batch) after
        # this call's last copy; `stream` is then that copy stream
        self._event = event

    def done(self) -> bool:
        return self._event.query() if self._event is not None else self.stream.query()

    def wait(self) -> None:
        """Block the host until this call's result is in ``out``."""
        if self._event is not None:
            self._event.synchronize()
        else:
            self.stream.synchronize()

    def result(self, with_stats: bool = False):
        """The (N, 2) host tensor of (u, v) rows once the call has finished.
        Raises :class:`OutOfDomainError` like :func:`evaluate_host` when a
        particle lay outside the domain (quadtree.py:191-198; the count rides
        along on the stream, no extra synchronisation).  ``with_stats=True``
        also returns the counters (vfmm_read_stats, no timings)."""
        self.wait()
        keep, self._keep = self._keep, None
        nbad = int(self._bad[0])
        if nbad:
            xs, ys = (k[0].numpy() if isinstance(k[0], torch.Tensor) else k[0] for k in keep[:2])
            bad = _bad_indices(xs, ys, self._domain)
            raise OutOfDomainError(
                f"{nbad} particle(s) outside domain {self._domain}, first indices {bad[:5].tolist()}"
            )
        if not with_stats:
            return self.out
        lib = _lib.load()
        st = _lib.VfmmStats()
        status = lib.vfmm_read_stats(self._n, self._config.levels, self._config.order, self._code,
                                     float(self._domain.side), self.ws.ptr, ctypes.byref(st),
                                     self.stream.cuda_stream)
        if status == _lib.VFMM_EDOMAIN:
            raise OutOfDomainError(f"particle(s) outside domain {self._domain}")
        _lib.check(status, "vfmm_read_stats")
        return self.out, _stats_from(st)


def _uniform_sigma(keep_entry):
    """The shared core size when every sigma is bitwise identical, else None."""
    obj = keep_entry[0]
    arr = obj.numpy() if isinstance(obj, torch.Tensor) else np.asarray(obj)
    if arr.size == 0:
        return None
    bits = torch.from_numpy(arr.reshape(-1).view(np.int64))
    lo, hi = torch.aminmax(bits)  # one pass, no temporary (numpy's ==/all took ~0.4 ms at N = 2^20)
    return float(arr.reshape(-1)[0]) if bool(lo == hi) else None


def evaluate_host_async(x, y, gamma, sigma, config, domain, *, out: torch.Tensor,
                        workspace: "Workspace", stream: torch.cuda.Stream, overlap: bool = True,
                        scalar_sigma: bool = True, graph: bool = True, copy_streams=None):
    """Asynchronous :func:`evaluate_host` (``vfmm_evaluate_host`` without
    VFMM_FLAG_STATS): enqueues the copies and the evaluation on ``stream`` and
    returns a :class:`PendingEvaluation` at once.  Calls on distinct streams
    and distinct workspaces pipeline -- the host<->device copies of one call
    overlap the compute of its neighbours -- which is how a batch of
    independent evaluations reaches the PCIe / compute bound instead of
    their sum.  ``x .. sigma`` and ``out`` must stay alive (and unchanged)
    until :meth:`PendingEvaluation.result`; pinned memory for full speed.
    With ``scalar_sigma`` a sigma array whose entries are all bitwise equal
    is sent as one value (VFMM_FLAG_SIGMA_SCALAR; the host check is hidden
    behind the previous evaluation's GPU work when calls are pipelined).
    With ``graph`` (default) the device part is one cached CUDA-graph launch
    per call (VFMM_FLAG_GRAPH; captured on the first call of each
    workspace / shape / domain).  ``copy_streams=(h2d, d2h)`` puts the input
    copies and the result copy on those two streams (shared by a batch) and
    only the graph on ``stream`` (``vfmm_evaluate_host_streams``): inputs
    then run ahead of the compute and results drain behind it."""
    validate_config(config)
    require_cuda()
    lib = _lib.load()
    keep = [_host_f64(a) for a in (x, y, gamma, sigma)]
    n = keep[0][0].numel() if isinstance(keep[0][0], torch.Tensor) else int(np.asarray(keep[0][0]).size)
    if n != workspace.n or config.levels != workspace.levels or config.order != workspace.order:
        raise ValueError("workspace shape does not match (n, levels, order)")
    if tuple(out.shape) != (n, 2) or not out.is_contiguous() or out.is_cuda:
        raise ValueError("out must be a contiguous host (N, 2) float64 tensor")
    code = kernel_code(config.kernel)
    flags = _lib.FLAG_UV_PAIRS | (_lib.FLAG_OVERLAP if overlap else 0) | (_lib.FLAG_GRAPH if graph else 0)
    sig_ptr = keep[3][1]
    if code == _lib.KERNEL_GAUSSIAN and scalar_sigma:
        one = _uniform_sigma(keep[3])
        if one is not None:
            # one pinned value per workspace (its previous call has completed
            # when the workspace is reused)
            scalar = getattr(workspace, "_sigma_scalar", None)
            if scalar is None:
                scalar = workspace._sigma_scalar = torch.empty(1, dtype=torch.float64).pin_memory()
            scalar[0] = one
            sig_ptr = scalar.data_ptr()
            flags |= _lib.FLAG_SIGMA_SCALAR
    sig_arg = sig_ptr if code == _lib.KERNEL_GAUSSIAN else None
    bad = getattr(workspace, "_bad_count", None)
    if bad is None:
        bad = workspace._bad_count = torch.zeros(1, dtype=torch.int32).pin_memory()
    if copy_streams is not None:
        h2d, d2h = copy_streams
        status = lib.vfmm_evaluate_host_streams(
            keep[0][1], keep[1][1], keep[2][1], sig_arg, n, float(domain.xmin), float(domain.ymin),
            float(domain.side), config.levels, config.order, code, out.data_ptr(), None, workspace.ptr,
            workspace.nbytes, flags, stream.cuda_stream, h2d.cuda_stream, d2h.cuda_stream,
        )
        _lib.check(status, "vfmm_evaluate_host_streams")
        _lib.check(lib.vfmm_bad_count_async(n, config.levels, config.order, workspace.ptr, bad.data_ptr(),
                                            d2h.cuda_stream), "vfmm_bad_count_async")
        event = getattr(workspace, "_done_event", None)
        if event is None:  # one call per workspace in flight: the event is reused
            event = workspace._done_event = torch.cuda.Event()
        event.record(d2h)
        return PendingEvaluation(out, d2h, keep, workspace, config, domain, n, code, bad, event)
    status = lib.vfmm_evaluate_host(
        keep[0][1], keep[1][1], keep[2][1], sig_arg, n,
        float(domain.xmin), float(domain.ymin), float(domain.side), config.levels, config.order,
        code, out.data_ptr(), None, workspace.ptr, workspace.nbytes, flags, None, stream.cuda_stream,
    )
    _lib.check(status, "vfmm_evaluate_host")
    _lib.check(lib.vfmm_bad_count_async(n, config.levels, config.order, workspace.ptr, bad.data_ptr(),
                                        stream.cuda_stream), "vfmm_bad_count_async")
    return PendingEvaluation(out, stream, keep, workspace, config, domain, n, code, bad)


class HostPipeline:
    """``depth`` evaluations of one (n, config, domain) shape in flight, each
    with its own workspace and pinned output buffer (round robin).

        pipe = HostPipeline(n, config, domain)
        pending = [pipe.submit(x, y, g, s) for (x, y, g, s) in batches]
        velocities = [p.result().clone() for p in pending]

    Three stages on three kinds of stream (``vfmm_evaluate_host_streams``):
    every call's input copies on ONE H2D stream, its cached CUDA graph on one
    of ``compute_streams`` streams (round robin: that many evaluations share
    the SMs, so the latency-bound head and tail of one hide behind the near
    field of another), its result copy on ONE D2H stream.  Input copies run
    ahead of the compute and results drain behind it: a batch runs at the
    slower of the PCIe copies and the overlapped compute.  With
    ``compute_streams=0`` every slot uses one stream for all three stages
    (the round-2 layout; A/B).  A slot's previous result is waited for before
    the slot is reused, so results must be consumed (copied) before ``depth``
    further submissions."""

    def __init__(self, n: int, config, domain, *, depth: int = 2, device=None, overlap: bool = True,
                 graph: bool = True, compute_streams: int | None = None):
        validate_config(config)
        require_cuda()
        dev = device_of(device)
        self.n, self.config, self.domain, self.overlap, self.graph = n, config, domain, overlap, graph
        if compute_streams is None:
            compute_streams = min(depth, 4) if graph else 0
        if compute_streams and not graph:
            raise ValueError("the three-stream pipeline replays CUDA graphs (graph=True)")
        self.copy_streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev)) if compute_streams else None
        self.compute = [torch.cuda.Stream(dev) for _ in range(compute_streams)]
        self.slots = [(Workspace(n, config.levels, config.order, dev), torch.cuda.Stream(dev),
                       torch.empty((n, 2), dtype=torch.float64, pin_memory=True)) for _ in range(depth)]
        self.pending = [None] * depth
        self.k = 0

    def submit(self, x, y, gamma, sigma) -> PendingEvaluation:
        i = self.k % len(self.slots)
        if self.pending[i] is not None:  # the slot's buffers must be free
            self.pending[i].wait()
        ws, stream, out = self.slots[i]
        if self.compute:
            stream = self.compute[self.k % len(self.compute)]
        self.k += 1
        self.pending[i] = evaluate_host_async(x, y, gamma, sigma, self.config, self.domain, out=out,
                                              workspace=ws, stream=stream, overlap=self.overlap,
                                              graph=self.graph, copy_streams=self.copy_streams)
        return self.pending[i]


def evaluate(
    particles: Sequence,
    config,
    domain=None,
    *,
    overlap: bool = True,
    timings: bool = False,
) -> tuple[np.ndarray, FmmRunStats]:
    """Velocity induced at every particle position, with run statistics (engine.py:335-398).

    Returns an (N, 2) float64 array of (u, v) rows in the original particle
    order.  When no domain is given, the smallest enclosing square is used.
    """
    validate_config(config)
    if len(particles) == 0:
        raise ValueError("need at least one particle")
    x, y, gamma, sigma = to_arrays(particles)
    if domain is None:
        domain = enclosing_domain_of(x, y)
    vel, stats = evaluate_host(x, y, gamma, sigma, config, domain, overlap=overlap, timings=timings,
                               stacklevel=3, out=torch.empty((len(x), 2), dtype=torch.float64))
    return vel.numpy(), stats


def evaluate_at(targets, particles: Sequence, config, domain=None) -> np.ndarray:
    """Velocity at arbitrary in-domain target points (engine.py:401-460)."""
    validate_config(config)
    x, y, gamma, sigma = to_arrays(particles)
    if domain is None:
        domain = enclosing_domain_of(x, y) if len(x) else Domain(0.0, 0.0, 1.0)
    pts = np.asarray(targets, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 2:
        raise ValueError(f"targets must have shape (M, 2), got {pts.shape}")
    inside = (
        (pts[:, 0] >= domain.xmin)
        & (pts[:, 0] <= domain.xmax)
        & (pts[:, 1] >= domain.ymin)
        & (pts[:, 1] <= domain.ymax)
    )
    if not inside.all():
        raise OutOfDomainError(f"{np.count_nonzero(~inside)} target(s) outside domain {domain}")
    u, v = evaluate_at_arrays(
        np.ascontiguousarray(pts[:, 0]), np.ascontiguousarray(pts[:, 1]),
        x, y, gamma, sigma, config, domain,
    )
    return np.stack((u.cpu().numpy(), v.cpu().numpy()), axis=1)


def evaluate_at_arrays(tx, ty, x, y, gamma, sigma, config, domain, *, device=None):
    """Device-array form of :func:`evaluate_at`; returns (u, v) CUDA tensors."""
    validate_config(config)
    require_cuda()
    lib = _lib.load()
    dev = device_of(device, tx, x)
    txd, tyd = as_device_f64(tx, dev), as_device_f64(ty, dev)
    m = int(txd.numel())
    u = torch.zeros(m, dtype=torch.float64, device=dev)
    v = torch.zeros(m, dtype=torch.float64, device=dev)
    xd, yd, gd = (as_device_f64(a, dev) for a in (x, y, gamma))
    n = int(xd.numel())
    if n == 0 or m == 0:
        return u, v
    code = kernel_code(config.kernel)
    sd = as_device_f64(sigma, dev) if code == _lib.KERNEL_GAUSSIAN else None
    ws = Workspace.get(n, config.levels, config.order, dev)
    st = _lib.VfmmStats()
    status = lib.vfmm_evaluate(
        xd.data_ptr(), yd.data_ptr(), gd.data_ptr(), sd.data_ptr() if sd is not None else None, n,
        float(domain.xmin), float(domain.ymin), float(domain.side), config.levels, config.order,
        code, None, None, ws.ptr, ws.nbytes, _lib.FLAG_STATS | _lib.FLAG_FAR_ONLY,
        ctypes.byref(st), stream_ptr(dev),
    )
    if status == _lib.VFMM_EDOMAIN:
        bad = _bad_indices(xd, yd, domain)
        raise OutOfDomainError(
            f"{bad.size} particle(s) outside domain {domain}, first indices {bad[:5].tolist()}"
        )
    _lib.check(status, "vfmm_evaluate(far only)")
    nbad = ctypes.c_int64(0)
    status = lib.vfmm_evaluate_at(
        txd.data_ptr(), tyd.data_ptr(), m, n, float(domain.xmin), float(domain.ymin),
        float(domain.side), config.levels, config.order, code, u.data_ptr(), v.data_ptr(), ws.ptr,
        ctypes.byref(nbad), stream_ptr(dev),
    )
    if status == _lib.VFMM_EDOMAIN:
        raise OutOfDomainError(f"{nbad.value} target(s) outside domain {domain}")
    _lib.check(status, "vfmm_evaluate_at")
    return u, v
