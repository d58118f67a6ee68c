"""Multi-GPU sharded evaluate: one process per GPU, leaves sharded in row strips.

SURVEY.md §8(e).  The leaf grid (2^l x 2^l, row-major keys) is cut into
``world`` contiguous strips of leaf rows, so a strip is a contiguous range of
leaf keys (the row-major analogue of a Morton range).  Per evaluate:

1. **redistribution** -- every particle goes to the rank owning its leaf row
   (``all_to_all_single``; the binning is the reference floor rule,
   quadtree.py:39-46, evaluated with the same IEEE operations as the kernel);
2. **particle halo** -- each rank sends the particles of its first / last owned
   row to the neighbour below / above, which is exactly what the P2P of its
   boundary leaves needs (3x3 neighbourhoods, engine.py:216-235);
3. **upward** on the GPU (``vfmm_evaluate_shard`` PHASE_UP), strip-local: P2M
   of the owned leaves, M2M of the subtrees touching the strip (partial
   multipoles for coarse cells straddling strips); the near field starts;
4. **multipole exchange** over NCCL (``exchange_multipoles``): an allgather of
   the small coarse levels 2..kc (each rank's partials, summed in rank order
   by ``vfmm_shard_unpack``) and a grouped send / recv with the neighbour
   strips of one plane row per parity plane of every fine level -- the two
   cell rows the M2L reaches beyond the strip (engine.py:77-89).  Config 3 on
   8 ranks: ~0.7 MB of multipoles per rank and direction instead of the
   117 MB pyramid;
5. **downward** on the GPU (PHASE_DOWN): M2L / L2L for cells touching the
   strip, P2P for owned leaves, L2P + combine for owned particles;
6. **counters** -- int64 all-reduce; each rank counts only what it owns, so the
   sums equal the single-GPU ``m2l_count`` / ``near_pair_count``.

The host orchestration is backend-agnostic: the CUDA backend calls the C ABI;
tests inject a CPU backend built on the oracle to check the decomposition on
``gloo`` (tests/test_distributed.py).  There is no silent fallback: the
default backend is CUDA and raises without a GPU.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from ._device import require_cuda, stream_ptr
from .engine import FmmRunStats, Workspace, validate_config
from .kernels import kernel_code
from .quadtree import OutOfDomainError


def row_bounds(levels: int, world: int) -> list[tuple[int, int]]:
    """Near-equal strips of the 2^levels leaf rows: rank r owns [b_r, b_{r+1}),
    b_r = floor(r m / world) rounded down to a multiple of u, the largest power
    of two <= m / (8 world) (1 for small grids).  Power-of-two worlds get
    exact equal strips; other worlds get strips within ~1/8 of each other
    whose boundaries sit on even cell rows of more levels, so fewer levels
    have to be all-gathered (``coarse_cut``)."""
    m = 2**levels
    u = 1
    while 2 * u <= m // (8 * world):
        u *= 2
    b = [(r * m // world) // u * u for r in range(world)] + [m]
    return [(b[r], b[r + 1]) for r in range(world)]


def leaf_rows(y: torch.Tensor, domain, levels: int) -> torch.Tensor:
    """Leaf row of each particle: min(int((y - ymin) / side * m), m - 1) (quadtree.py:44-45)."""
    m = 2**levels
    return torch.clamp(((y - domain.ymin) / domain.side * m).to(torch.int64), max=m - 1)


def owner_of_rows(rows: torch.Tensor, bounds) -> torch.Tensor:
    starts = torch.tensor([lo for lo, _ in bounds], dtype=torch.int64, device=rows.device)
    return torch.searchsorted(starts, rows, right=True) - 1


def coarse_cut(levels: int, bounds) -> int:
    """kc: the levels 2..kc are all-gathered, the levels above exchange halo rows.

    A level k is "fine" when every non-empty strip starts and ends on an even
    cell row of level k and is at least two cell rows tall: the two cell rows
    the M2L reaches beyond a strip then belong to the neighbour strip and form
    one row of each parity plane.  Fine levels are closed upwards, so kc is
    the finest level that is not fine (1 when every level is)."""
    kc = 1
    for k in range(2, levels + 1):
        sft = levels - k
        mask = (1 << (sft + 1)) - 1
        fine = all((lo & mask) == 0 and (hi & mask) == 0 and ((hi - lo) >> sft) >= 2
                   for lo, hi in bounds if hi > lo)
        if not fine:
            kc = k
    return kc


def neighbours(bounds, rank: int):
    """(rank below, rank above) of a strip: the nearest ranks with non-empty strips."""
    if bounds[rank][1] <= bounds[rank][0]:
        return None, None
    below = next((r for r in range(rank - 1, -1, -1) if bounds[r][1] > bounds[r][0]), None)
    above = next((r for r in range(rank + 1, len(bounds)) if bounds[r][1] > bounds[r][0]), None)
    return below, above


def _exchange(cols: torch.Tensor, dest: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Send column j of ``cols`` [k, n] to rank dest[j]; returns the received [k, n'] in
    (source rank, original position) order."""
    order = torch.argsort(dest, stable=True)
    send = cols[:, order].t().contiguous()  # [n, k] rows grouped by destination
    counts = torch.bincount(dest, minlength=world).to(torch.int64)
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts, group=group)
    k = cols.shape[0]
    recv = torch.empty((int(recv_counts.sum()), k), dtype=cols.dtype, device=cols.device)
    dist.all_to_all_single(recv, send, output_split_sizes=recv_counts.tolist(),
                           input_split_sizes=counts.tolist(), group=group)
    return recv.t().contiguous()


@dataclass
class Shard:
    """This rank's particles after redistribution: owned first, then halo."""

    cols: torch.Tensor  # [5, n_local] float64: x, y, gamma, sigma, global id
    n_owned: int
    rows: tuple[int, int]


def redistribute_owned(x, y, gamma, sigma, ids, domain, levels: int, group=None):
    """Step 1: every particle to the rank owning its leaf row.  Returns the
    owned columns [5, n_owned] (x, y, gamma, sigma, global id) and the strip."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    bounds = row_bounds(levels, world)
    cols = torch.stack([x, y, gamma, sigma, ids.to(torch.float64)])
    owned = _exchange(cols, owner_of_rows(leaf_rows(cols[1], domain, levels), bounds), world, group)
    return owned, bounds[rank]


def add_halo(owned: torch.Tensor, rows, domain, levels: int, group=None) -> Shard:
    """Step 2: my first owned leaf row goes to the strip below, my last to the
    strip above (grouped NCCL send / recv with the two neighbours).  One host
    synchronisation: the four message sizes, read together, size the receive
    buffers; the compaction uses ``nonzero_static`` (no further syncs)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    bounds = row_bounds(levels, world)
    lo, hi = rows
    below, above = neighbours(bounds, rank)
    glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    r = leaf_rows(owned[1], domain, levels)
    dev = owned.device
    m_down = (r == lo) if below is not None else torch.zeros_like(r, dtype=torch.bool)
    m_up = (r == hi - 1) if above is not None else torch.zeros_like(r, dtype=torch.bool)
    sizes = torch.stack([m_down.sum(), m_up.sum()]).to(torch.int64)
    recv_sizes = torch.zeros(2, dtype=torch.int64, device=dev)  # from below, from above
    ops = []
    if below is not None:
        ops += [dist.P2POp(dist.isend, sizes[0:1].contiguous(), glob(below), group),
                dist.P2POp(dist.irecv, recv_sizes[0:1], glob(below), group)]
    if above is not None:
        ops += [dist.P2POp(dist.isend, sizes[1:2].contiguous(), glob(above), group),
                dist.P2POp(dist.irecv, recv_sizes[1:2], glob(above), group)]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    n_down, n_up, n_below, n_above = torch.cat([sizes, recv_sizes]).tolist()  # the one sync
    k = owned.shape[0]
    send_down = owned[:, torch.nonzero_static(m_down, size=n_down).flatten()].contiguous()
    send_up = owned[:, torch.nonzero_static(m_up, size=n_up).flatten()].contiguous()
    from_below = torch.empty((k, n_below), dtype=owned.dtype, device=dev)
    from_above = torch.empty((k, n_above), dtype=owned.dtype, device=dev)
    ops = []
    if below is not None:
        ops += [dist.P2POp(dist.isend, send_down, glob(below), group),
                dist.P2POp(dist.irecv, from_below, glob(below), group)]
    if above is not None:
        ops += [dist.P2POp(dist.isend, send_up, glob(above), group),
                dist.P2POp(dist.irecv, from_above, glob(above), group)]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return Shard(torch.cat([owned, from_below, from_above], dim=1), owned.shape[1], (lo, hi))


def redistribute(x, y, gamma, sigma, ids, domain, levels: int, group=None) -> Shard:
    """Steps 1-2: owner redistribution and one-row halo exchange."""
    owned, rows = redistribute_owned(x, y, gamma, sigma, ids, domain, levels, group)
    return add_halo(owned, rows, domain, levels, group)


class CudaShardBackend:
    """PHASE_UP / PHASE_DOWN of ``vfmm_evaluate_shard`` on this rank's GPU."""

    def __init__(self, device: torch.device, private_workspace: bool = False,
                 up_flags: int = _lib.FLAG_OVERLAP, down_flags: int = _lib.FLAG_OVERLAP):
        require_cuda()
        self.device = device
        self.private = private_workspace
        self.up_flags, self.down_flags = up_flags, down_flags
        self.lib = _lib.load()
        self.ws = None

    def _args(self, shard: Shard, config, domain):
        c = shard.cols
        return (c[0].data_ptr(), c[1].data_ptr(), c[2].data_ptr(), c[3].data_ptr(), c.shape[1],
                float(domain.xmin), float(domain.ymin), float(domain.side), config.levels,
                config.order, kernel_code(config.kernel), shard.rows[0], shard.rows[1])

    def up(self, shard: Shard, config, domain):
        """PHASE_UP (asynchronous on the current stream); OVERLAP starts the near field."""
        nl = shard.cols.shape[1]
        self.shape = (nl, config.levels, config.order, shard.rows)
        if nl == 0:
            self.ws = None
            return
        self.ws = (Workspace(nl, config.levels, config.order, self.device) if self.private
                   else Workspace.get(nl, config.levels, config.order, self.device))
        rc = self.lib.vfmm_evaluate_shard(*self._args(shard, config, domain), None, None,
                                          self.ws.ptr, self.ws.nbytes,
                                          _lib.FLAG_PHASE_UP | self.up_flags, None,
                                          stream_ptr(self.device))
        _lib.check(rc, "vfmm_evaluate_shard(up)")

    def _buffers(self, kc: int):
        """Exchange buffers (reused across calls: graph replays see fixed addresses)."""
        nl, lv, p, (lo, hi) = self.shape
        key = (lv, p, lo, hi, kc)
        if getattr(self, "_buf_key", None) != key:
            cb, hb = ctypes.c_size_t(), ctypes.c_size_t()
            rc = self.lib.vfmm_shard_exchange_size(max(nl, 1), lv, p, lo, hi, kc, ctypes.byref(cb),
                                                   ctypes.byref(hb))
            _lib.check(rc, "vfmm_shard_exchange_size")
            mk = lambda b: torch.zeros(b, dtype=torch.uint8, device=self.device)  # noqa: E731
            self._bufs = {"coarse": mk(cb.value), "down": mk(hb.value), "up": mk(hb.value),
                          "below": mk(hb.value), "above": mk(hb.value)}
            self._buf_key = key
        return self._bufs

    def pack(self, kc: int, below: bool, above: bool):
        """(coarse contribution, rows for the strip below, rows for the strip above);
        byte tensors, None where there is nothing to send."""
        nl, lv, p, (lo, hi) = self.shape
        b = self._buffers(kc)
        coarse = b["coarse"] if b["coarse"].numel() else None
        down = b["down"] if below and b["down"].numel() else None
        up = b["up"] if above and b["up"].numel() else None
        if self.ws is None:  # nothing local: a zero contribution
            if coarse is not None:
                coarse.zero_()
            return coarse, down, up
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        rc = self.lib.vfmm_shard_pack(nl, lv, p, lo, hi, kc, self.ws.ptr, ptr(coarse), ptr(down),
                                      ptr(up), stream_ptr(self.device))
        _lib.check(rc, "vfmm_shard_pack")
        return coarse, down, up

    def recv_buffers(self, kc: int):
        b = self._buffers(kc)
        return b["below"], b["above"]

    def unpack(self, kc: int, coarse_all, world: int, from_below, from_above):
        if self.ws is None:
            return
        nl, lv, p, (lo, hi) = self.shape
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        rc = self.lib.vfmm_shard_unpack(nl, lv, p, lo, hi, kc, self.ws.ptr, ptr(coarse_all), world,
                                        ptr(from_below), ptr(from_above), stream_ptr(self.device))
        _lib.check(rc, "vfmm_shard_unpack")

    def down(self, shard: Shard, config, domain, counters: bool = True):
        """(2, n_local) velocities (owned columns valid), m2l_count, near_pair_count
        (the counters cost a stream synchronisation; 0, 0 when not requested)."""
        n = shard.cols.shape[1]
        vel = torch.zeros((2, n), dtype=torch.float64, device=self.device)
        if n == 0:
            return vel, 0, 0
        rc = self.lib.vfmm_evaluate_shard(*self._args(shard, config, domain), vel[0].data_ptr(),
                                          vel[1].data_ptr(), self.ws.ptr, self.ws.nbytes,
                                          _lib.FLAG_PHASE_DOWN | self.down_flags, None,
                                          stream_ptr(self.device))
        _lib.check(rc, "vfmm_evaluate_shard(down)")
        if not counters:
            return vel, 0, 0
        st = _lib.VfmmStats()
        rc = self.lib.vfmm_read_stats(n, config.levels, config.order, kernel_code(config.kernel),
                                      float(domain.side), self.ws.ptr, ctypes.byref(st),
                                      stream_ptr(self.device))
        _lib.check(rc, "vfmm_read_stats")
        return vel, int(st.m2l_count), int(st.near_pair_count)


def _all_gather_bytes(out: torch.Tensor, inp: torch.Tensor, world: int, group=None):
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
    else:
        dist.all_gather(list(out.view(world, -1).unbind(0)), inp, group=group)


def exchange_multipoles(backend, config, world: int, rank: int, group=None, stats: dict | None = None):
    """Step 4: coarse allgather + neighbour halo rows, between PHASE_UP and PHASE_DOWN."""
    bounds = row_bounds(config.levels, world)
    kc = coarse_cut(config.levels, bounds)
    below, above = neighbours(bounds, rank)
    coarse, down, up = backend.pack(kc, below is not None, above is not None)
    coarse_all = None
    if coarse is not None:
        coarse_all = torch.empty(world * coarse.numel(), dtype=torch.uint8, device=coarse.device)
        _all_gather_bytes(coarse_all, coarse, world, group)
    rb, ra = backend.recv_buffers(kc)
    from_below = rb if down is not None else None
    from_above = ra if up is not None else None
    ops = []
    glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    if below is not None and down is not None:
        ops += [dist.P2POp(dist.isend, down, glob(below), group),
                dist.P2POp(dist.irecv, from_below, glob(below), group)]
    if above is not None and up is not None:
        ops += [dist.P2POp(dist.isend, up, glob(above), group),
                dist.P2POp(dist.irecv, from_above, glob(above), group)]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    backend.unpack(kc, coarse_all, world, from_below, from_above)
    if stats is not None:
        stats.update(kc=kc, coarse_bytes=0 if coarse is None else coarse.numel(),
                     halo_bytes_sent=sum(t.numel() for t in (down, up) if t is not None),
                     recv_bytes=(0 if coarse_all is None else coarse_all.numel())
                     + sum(t.numel() for t in (from_below, from_above) if t is not None))


def evaluate_shard(shard: Shard, config, domain, *, backend=None, group=None, counters=True):
    """Steps 3-6 on a prepared shard: upward, multipole exchange, downward, counters.
    Returns ((2, n_local) velocities, FmmRunStats or None)."""
    if backend is None:
        backend = CudaShardBackend(shard.cols.device)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    backend.up(shard, config, domain)
    exchange_multipoles(backend, config, world, rank, group)
    vel, m2l, near = backend.down(shard, config, domain, counters=counters)
    if not counters:
        return vel, None
    cnt = torch.tensor([m2l, near, shard.n_owned], dtype=torch.int64, device=shard.cols.device)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    return vel, FmmRunStats(n=int(cnt[2]), levels=config.levels, order=config.order,
                            m2l_count=int(cnt[0]), near_pair_count=int(cnt[1]))


def evaluate_sharded(x, y, gamma, sigma, ids, config, domain, *, backend=None, group=None):
    """Sharded evaluate on this rank's input slice.

    ``x, y, gamma, sigma, ids`` are this rank's input particles (any subset of
    the global set; ``ids`` are their global indices).  Returns
    ``(owned_ids, vel, stats)``: the global ids of the particles this rank now
    owns, their (2, n_owned) velocities and the global ``FmmRunStats`` counters.
    """
    validate_config(config)
    if backend is None:
        backend = CudaShardBackend(x.device)
    inside = (x >= domain.xmin) & (x <= domain.xmax) & (y >= domain.ymin) & (y <= domain.ymax)
    bad = torch.tensor([int((~inside).sum())], dtype=torch.int64, device=x.device)
    dist.all_reduce(bad, group=group)
    if int(bad):
        raise OutOfDomainError(f"{int(bad)} particle(s) outside domain {domain}")
    shard = redistribute(x, y, gamma, sigma, ids, domain, config.levels, group)
    vel, stats = evaluate_shard(shard, config, domain, backend=backend, group=group)
    k = shard.n_owned
    return shard.cols[4, :k].to(torch.int64), vel[:, :k], stats


def gather_velocities(owned_ids, vel, n_total: int, group=None, dst: int = 0):
    """Assemble the (N, 2) velocities in global order on rank ``dst`` (None elsewhere)."""
    world = dist.get_world_size(group)
    cnt = torch.tensor([owned_ids.numel()], dtype=torch.int64, device=vel.device)
    sizes = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(sizes, cnt, group=group)
    mx = max(int(s) for s in sizes)
    pad = torch.zeros((3, mx), dtype=torch.float64, device=vel.device)
    pad[0, : owned_ids.numel()] = owned_ids.to(torch.float64)
    pad[1:, : owned_ids.numel()] = vel
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if dist.get_rank(group) != dst:
        return None
    out = torch.empty((n_total, 2), dtype=torch.float64, device=vel.device)
    for s, b in zip(sizes, bufs):
        k = int(s)
        out[b[0, :k].to(torch.int64)] = b[1:, :k].t()
    return out


def make_shards(x, y, gamma, sigma, domain, levels: int, world: int) -> list[Shard]:
    """The shards ``redistribute`` produces, built locally for ``world`` logical ranks."""
    bounds = row_bounds(levels, world)
    rows = leaf_rows(y, domain, levels)
    owner = owner_of_rows(rows, bounds)
    ids = torch.arange(x.numel(), device=x.device)
    m = 2**levels
    shards = []
    for r, (lo, hi) in enumerate(bounds):
        own = torch.nonzero(owner == r).flatten()
        below = torch.nonzero((rows == lo - 1) & (lo > 0) & (hi > lo)).flatten()
        above = torch.nonzero((rows == hi) & (hi < m) & (hi > lo)).flatten()
        idx = torch.cat([own, below, above])
        cols = torch.stack([x[idx], y[idx], gamma[idx], sigma[idx], ids[idx].to(torch.float64)])
        shards.append(Shard(cols.contiguous(), own.numel(), (lo, hi)))
    return shards


def evaluate_emulated(x, y, gamma, sigma, config, domain, world: int, backend_factory=None):
    """``world`` logical ranks run one after another on one device, with the
    exchange done locally: every rank's PHASE_UP and pack, the coarse
    contributions concatenated and every rank's unpack with its neighbours'
    halo rows, then every rank's PHASE_DOWN.  Exercises the row-restricted kernels of the
    sharded path on a single GPU (R logical ranks sequentially).
    Returns ((2, N) velocities, m2l_count, near_pair_count)."""
    validate_config(config)
    if backend_factory is None:
        def backend_factory():
            return CudaShardBackend(x.device, private_workspace=True)
    shards = make_shards(x, y, gamma, sigma, domain, config.levels, world)
    backends = [backend_factory() for _ in shards]
    for b, sh in zip(backends, shards):
        b.up(sh, config, domain)
    bounds = row_bounds(config.levels, world)
    kc = coarse_cut(config.levels, bounds)
    nb = [neighbours(bounds, r) for r in range(world)]
    packs = [b.pack(kc, lo is not None, hi is not None) for b, (lo, hi) in zip(backends, nb)]
    coarse_all = (torch.cat([p[0] for p in packs]) if packs and packs[0][0] is not None else None)
    for r, b in enumerate(backends):
        below, above = nb[r]
        b.unpack(kc, coarse_all, world, packs[below][2] if below is not None else None,
                 packs[above][1] if above is not None else None)
    out = torch.zeros((2, x.numel()), dtype=torch.float64, device=x.device)
    m2l = near = 0
    for sh, b in zip(shards, backends):
        vel, c1, c2 = b.down(sh, config, domain)
        m2l += c1
        near += c2
        k = sh.n_owned
        out[:, sh.cols[4, :k].to(torch.int64)] = vel[:, :k]
    return out, m2l, near


# ----------------------------------------------------------------------------- bench
def e2e_loop(variant, host_cols, owned, rows_in, rows, dom, cfg, backend, steps, dev):
    """ms per step of the multi-GPU bench's end-to-end loop: every step copies
    this rank's inputs (the first ``rows_in`` rows of the owned columns) in
    from pinned host memory, exchanges the particle halo, runs the sharded
    evaluate and copies the owned velocities out.  "copy" (default): two
    steps in flight, inputs and outputs on a copy stream; "sync": one step at
    a time (A/B).  Two untimed steps first."""
    main = torch.cuda.Stream(dev)
    with torch.cuda.stream(main):
        _e2e_loop(variant, host_cols, owned, rows_in, rows, dom, cfg, backend, 2, dev, main)
        return _e2e_loop(variant, host_cols, owned, rows_in, rows, dom, cfg, backend, steps, dev, main)


def _e2e_loop(variant, host_cols, owned, rows_in, rows, dom, cfg, backend, steps, dev, main):
    import time

    k_own = owned.shape[1]
    host_vel = [torch.empty((2, k_own), dtype=torch.float64).pin_memory() for _ in range(2)]
    dcols = [owned.clone() for _ in range(2)]  # resident sigma / id rows
    copy = torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = time.perf_counter()
    if variant == "sync":
        for _ in range(steps):
            dcols[0][:rows_in].copy_(host_cols[:rows_in], non_blocking=True)
            sh = add_halo(dcols[0], rows, dom, cfg.levels)
            vel, _ = evaluate_shard(sh, cfg, dom, backend=backend, counters=False)
            host_vel[0].copy_(vel[:, :k_own], non_blocking=True)
            torch.cuda.synchronize(dev)
        return (time.perf_counter() - t0) * 1e3 / steps
    with torch.cuda.stream(copy):
        dcols[0][:rows_in].copy_(host_cols[:rows_in], non_blocking=True)
        ev_in[0].record(copy)
    for k in range(steps):
        b = k & 1
        main.wait_event(ev_in[b])
        if k + 1 < steps:  # the next step's inputs, once step k - 1 is done with the buffer
            if k >= 1:
                copy.wait_event(ev_used[b ^ 1])
            with torch.cuda.stream(copy):
                dcols[b ^ 1][:rows_in].copy_(host_cols[:rows_in], non_blocking=True)
                ev_in[b ^ 1].record(copy)
        sh = add_halo(dcols[b], rows, dom, cfg.levels)
        vel, _ = evaluate_shard(sh, cfg, dom, backend=backend, counters=False)
        ev_used[b].record(main)
        if k >= 2:
            ev_done[b].synchronize()  # the host buffer of step k - 2 is free
        vel.record_stream(copy)
        with torch.cuda.stream(copy):
            copy.wait_event(ev_used[b])
            host_vel[b].copy_(vel[:, :k_own], non_blocking=True)
            ev_done[b].record(copy)
    torch.cuda.synchronize(dev)
    return (time.perf_counter() - t0) * 1e3 / steps


def bench_main(args):
    """``bench.py --gpus N`` under torchrun: the sharded evaluate of a BASELINE config.

    Setup (untimed, as the single-GPU bench keeps its inputs resident): every
    rank generates the same seeded workload, sends its contiguous 1/N slice of
    the particles to their row-strip owners and exchanges the one-row halos.
    A step is the sharded evaluate -- PHASE_UP (tree, strip-local P2M / M2M;
    the near field starts), the multipole exchange (NCCL allgather of the
    coarse levels + grouped send / recv of the neighbours' halo rows),
    PHASE_DOWN (M2L, L2L, L2P + combine) -- captured in one CUDA graph and
    replayed with L2 flushed between steps; CUDA events between barriers, max
    over ranks.  ``e2e``: per step each rank copies its owned particles in
    from pinned host memory, exchanges the particle halo with its neighbours
    (one host synchronisation for the message sizes), runs the sharded
    evaluate and copies its velocities back; wall clock between barriers, max
    over ranks.
    """
    import json
    import time

    from . import workloads as W
    from .engine import FmmConfig
    from .kernels import KernelKind
    from .model import Domain

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # rank 0 prints ONE JSON line on stdout: NCCL's version banner (printed
    # when the first communicator comes up) goes to stderr instead
    import sys as _sys
    _sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
        torch.cuda.synchronize(dev)
    finally:
        _sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    w = W.by_index(args.config)
    cfg = FmmConfig(w.levels, w.order, KernelKind.GAUSSIAN_BLOB)
    dom = Domain(*W.DOMAIN)
    lib = _lib.load()
    lo, hi = rank * w.n // world, (rank + 1) * w.n // world
    x, y, g, s = (torch.from_numpy(a[lo:hi]).to(dev) for a in (w.x, w.y, w.gamma, w.sigma))
    ids = torch.arange(lo, hi, device=dev)
    owned, rows = redistribute_owned(x, y, g, s, ids, dom, cfg.levels)
    shard = add_halo(owned, rows, dom, cfg.levels)
    backend = CudaShardBackend(dev)
    _, st = evaluate_shard(shard, cfg, dom, backend=backend, counters=True)
    xstat = {}
    backend.up(shard, cfg, dom)  # one more step, recording the exchange sizes
    exchange_multipoles(backend, cfg, world, rank, stats=xstat)
    backend.down(shard, cfg, dom, counters=False)
    xs = torch.tensor([xstat.get("recv_bytes", 0), xstat.get("halo_bytes_sent", 0)], dtype=torch.int64,
                      device=dev)
    dist.all_reduce(xs, op=dist.ReduceOp.MAX)
    xstat = {"coarse_levels": f"2..{xstat.get('kc', 1)}" if xstat.get("kc", 1) >= 2 else "none",
             "max_recv_bytes_per_rank": int(xs[0]), "max_halo_bytes_sent_per_rank": int(xs[1])}

    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            evaluate_shard(shard, cfg, dom, backend=backend, counters=False)
    torch.cuda.synchronize(dev)
    c0 = lib.vfmm_launch_count()
    graph = torch.cuda.CUDAGraph()
    mode = "CUDA graph replay"
    try:  # NCCL collectives and grouped send / recv are graph-capturable
        with torch.cuda.graph(graph, stream=stream):
            evaluate_shard(shard, cfg, dom, backend=backend, counters=False)
        replay = graph.replay
    except Exception as exc:  # pragma: no cover - depends on the NCCL / torch build
        torch.cuda.synchronize(dev)
        dist.barrier()
        mode = f"stream launches (graph capture failed: {type(exc).__name__})"

        def replay():
            evaluate_shard(shard, cfg, dom, backend=backend, counters=False)
    launches = lib.vfmm_launch_count() - c0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(max(3, args.warmup)):
        flush.zero_()
        replay()
    torch.cuda.synchronize(dev)
    dist.barrier()
    cur = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler = getattr(args, "clock_sampler", None)
    clk = sampler(local) if sampler is not None else None
    if clk is not None:
        clk.__enter__()
    for a, b in ev:
        flush.zero_()
        a.record(cur)
        replay()
        b.record(cur)
    torch.cuda.synchronize(dev)
    if clk is not None:
        clk.__exit__(None, None, None)
    dist.barrier()
    ms = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)

    # end to end from pinned host buffers (e2e_loop): owned particles in,
    # owned velocities out, every step, two steps in flight
    host_cols = owned.cpu().pin_memory()
    k_own = owned.shape[1]
    # the step's inputs: x, y, gamma -- and sigma unless every core size is
    # the same (then it travels as the resident column, like the single-GPU
    # path's one-value sigma); the global ids are the sharding's metadata and
    # stay resident
    sig = host_cols[3]
    sig_uniform = bool(k_own == 0 or bool((sig == sig[0]).all()))
    rows_in = int(os.environ.get("VFMM_E2E_ROWS", 3 if sig_uniform else 4))  # (env: A/B)
    h2d_row_bytes = 8 * rows_in
    e2e_steps = max(12, args.e2e_steps)  # two in flight: enough steps to amortise the fill
    variant = os.environ.get("VFMM_E2E_VARIANT", "copy")
    ms_e2e = e2e_loop(variant, host_cols, owned, rows_in, rows, dom, cfg, backend, e2e_steps, dev)
    e2e = torch.tensor([ms_e2e], device=dev)
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    nb = torch.tensor([owned.shape[1]], dtype=torch.int64, device=dev)
    dist.all_reduce(nb, op=dist.ReduceOp.MAX)

    # roofline of the dominant kernel (P2P) per rank: one extra sharded evaluate
    # in stats mode (phase events), achieved = 42 flop x this rank's near pairs /
    # its near-field time; the line reports the slowest rank
    roof = None
    peak_fn = getattr(args, "fp64_peak", None)
    if peak_fn is not None:
        import ctypes

        sh_vel = torch.zeros((2, shard.cols.shape[1]), dtype=torch.float64, device=dev)
        backend.up(shard, cfg, dom)
        backend.down(shard, cfg, dom, counters=False)
        torch.cuda.synchronize(dev)
        st_up, st_dn = _lib.VfmmStats(), _lib.VfmmStats()
        for ph, st_ in ((_lib.FLAG_PHASE_UP, st_up), (_lib.FLAG_PHASE_DOWN, st_dn)):
            rc = lib.vfmm_evaluate_shard(*backend._args(shard, cfg, dom), sh_vel[0].data_ptr(),
                                         sh_vel[1].data_ptr(), backend.ws.ptr, backend.ws.nbytes,
                                         ph | _lib.FLAG_OVERLAP | _lib.FLAG_STATS | _lib.FLAG_PHASE_TIMES,
                                         ctypes.byref(st_), stream_ptr(dev))
            _lib.check(rc, "vfmm_evaluate_shard(stats)")
        t_near = float(st_up.t_near) * 1e-3  # s (the near field runs in PHASE_UP)
        pairs = float(st_dn.near_pair_count)
        ach = 42.0 * pairs / t_near / 1e12 if t_near > 0 else 0.0
        peak = float(peak_fn(lib, torch, dev))
        rr = torch.tensor([ach, peak, t_near * 1e3], dtype=torch.float64, device=dev)
        gathered = [torch.zeros_like(rr) for _ in range(world)]
        dist.all_gather(gathered, rr)
        slow = min(gathered, key=lambda t: float(t[0]))
        roof = {"bound": "fp64", "kernel": "k_p2p (near field), slowest rank",
                "achieved": float(slow[0]), "peak": float(slow[1]), "unit": "TFLOP/s",
                "frac": float(slow[0] / slow[1]) if float(slow[1]) > 0 else None,
                "peak_source": "measured live: DFMA probe (vfmm_fp64_probe), per rank",
                "traffic": None, "p2p_ms": float(slow[2]), "flop_per_pair": 42}
    if rank == 0:
        print(json.dumps({
            "metric": "FMM particle velocity evals/sec (fp64)", "value": w.n / (float(ms) * 1e-3),
            "unit": "particle-evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(ms), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n": w.n, "levels": w.levels, "order": w.order,
                       "sharding": f"{world} row strips of leaves (+ one-row particle halos)",
                       "graph": f"{mode} of the sharded evaluate (PHASE_UP, NCCL "
                                "coarse-level allgather + neighbour halo-row send/recv of the "
                                "multipoles, PHASE_DOWN)",
                       "exchange": xstat,
                       "l2": "flushed between steps (256 MiB write)",
                       "m2l_count": st.m2l_count, "near_pair_count": st.near_pair_count},
            "e2e": {"value": w.n / (float(e2e) * 1e-3), "unit": "particle-evals/s",
                    "h2d_bytes_per_step": h2d_row_bytes * int(nb), "d2h_bytes_per_step": 16 * int(nb),
                    "ms_per_step": float(e2e),
                    "mode": "per rank: owned particles H2D, halo exchange, sharded evaluate, "
                            "velocities D2H, two steps in flight (copies on a copy stream); "
                            "wall clock, max over ranks (bytes: largest rank)"},
            "gpu_launches": int(launches) * args.steps,
            "roofline": roof, "cpu_baseline": None,
            "clocks": clk.summary() if clk is not None else None,
        }), flush=True)
    dist.destroy_process_group()
