"""Multi-GPU path on CPU: world-size-2 ``gloo`` runs of the
sharded orchestration (redistribution, halo exchange, multipole + occupancy
all-reduce, counter reduction, gather) with the oracle shard backend, checked
against the single-process oracle; plus logical-rank emulation for 1..8 strips
and the GPU shard kernels (``-m gpu``) against the single-GPU evaluate."""
import json
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_0809_1810_b200 as vf
from paper_0809_1810_b200 import distributed as D
from oracle import fmm_oracle as O
from _oracle_shard import OracleShardBackend

G = vf.KernelKind.GAUSSIAN_BLOB


def case(n=1500, seed=3, lattice=False):
    rng = np.random.default_rng(seed)
    if lattice:
        m = int(round(np.sqrt(n)))
        c = (np.arange(m) + 0.5) / m
        gx, gy = np.meshgrid(c, c)
        x, y = gx.ravel().copy(), gy.ravel().copy()
        # particles exactly on strip / leaf boundaries and on the max edges
        x[:5] = [0.0, 0.25, 0.5, 1.0, 0.75]
        y[:5] = [0.5, 0.25, 1.0, 0.0, 0.5]
    else:
        x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    g = rng.uniform(-1, 1, x.size)
    s = np.full(x.size, 0.004)
    return x, y, g, s


def _worker(rank, world, port, out_path, levels, order, lattice):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, y, g, s = case(lattice=lattice)
    ids = np.arange(x.size)
    mine = ids % world == rank  # interleaved input: redistribution moves most particles
    t = [torch.from_numpy(np.ascontiguousarray(a[mine])) for a in (x, y, g, s)]
    cfg = vf.FmmConfig(levels, order, G)
    dom = vf.Domain(0.0, 0.0, 1.0)
    own_ids, vel, st = D.evaluate_sharded(*t, torch.from_numpy(ids[mine]), cfg, dom,
                                          backend=OracleShardBackend())
    full = D.gather_velocities(own_ids, vel, x.size)
    if rank == 0:
        ref, rst = O.evaluate(x, y, g, s, levels, order, True, (0.0, 0.0, 1.0))
        err = float(np.abs(full.numpy() - ref).max() / np.abs(ref).max())
        json.dump({"err": err, "m2l": st.m2l_count, "m2l_ref": rst["m2l_count"],
                   "near": st.near_pair_count, "near_ref": rst["near_pair_count"], "n": st.n,
                   "n_ref": int(x.size)},
                  open(out_path, "w"))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("levels,order,lattice", [(4, 8, False), (3, 10, True)])
def test_gloo_world2_matches_single_process_oracle(levels, order, lattice):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.json")
        mp.spawn(_worker, args=(2, _free_port(), out, levels, order, lattice), nprocs=2, join=True)
        r = json.load(open(out))
    assert r["m2l"] == r["m2l_ref"] and r["near"] == r["near_ref"] and r["n"] == r["n_ref"]
    assert r["err"] <= 1e-13


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_logical_ranks_match_single_process_oracle(world):
    x, y, g, s = case(n=900, seed=world)
    cfg = vf.FmmConfig(3, 9, G)
    dom = vf.Domain(0.0, 0.0, 1.0)
    t = [torch.from_numpy(a) for a in (x, y, g, s)]
    vel, m2l, near = D.evaluate_emulated(*t, cfg, dom, world, backend_factory=OracleShardBackend)
    ref, rst = O.evaluate(x, y, g, s, 3, 9, True, (0.0, 0.0, 1.0))
    assert m2l == rst["m2l_count"] and near == rst["near_pair_count"]
    assert np.abs(vel.numpy().T - ref).max() <= 1e-13 * np.abs(ref).max()


def test_row_bounds_and_owner():
    b = D.row_bounds(3, 3)
    assert b == [(0, 2), (2, 5), (5, 8)]
    rows = torch.tensor([0, 1, 2, 4, 5, 7])
    assert D.owner_of_rows(rows, b).tolist() == [0, 0, 1, 1, 2, 2]
    assert D.row_bounds(2, 8)[0] == (0, 0)  # more ranks than rows: empty strips


def test_coarse_cut_and_neighbours():
    assert D.coarse_cut(7, D.row_bounds(7, 1)) == 1  # one strip: nothing to exchange
    assert D.coarse_cut(7, D.row_bounds(7, 2)) == 1  # every level fine: halo rows only
    assert D.coarse_cut(7, D.row_bounds(7, 4)) == 2
    assert D.coarse_cut(7, D.row_bounds(7, 8)) == 3
    assert D.coarse_cut(9, D.row_bounds(9, 8)) == 3
    b3 = D.row_bounds(7, 3)
    assert b3 == [(0, 40), (40, 84), (84, 128)] and D.coarse_cut(7, b3) == 5
    assert D.neighbours(D.row_bounds(7, 4), 0) == (None, 1)
    assert D.neighbours(D.row_bounds(7, 4), 3) == (2, None)
    b = D.row_bounds(2, 8)  # 4 rows, 8 ranks: empty strips are skipped
    assert D.neighbours(b, 2) == (None, None) or b[2][0] < b[2][1]
    nonempty = [r for r in range(8) if b[r][1] > b[r][0]]
    for i, r in enumerate(nonempty):
        lo, hi = D.neighbours(b, r)
        assert lo == (nonempty[i - 1] if i else None)
        assert hi == (nonempty[i + 1] if i + 1 < len(nonempty) else None)


def test_multipole_exchange_volume_config3_on_8_ranks():
    """SURVEY.md §8e / north_star: coarse allgather + neighbour halo rows instead of
    the whole pyramid (117 MB at config 3): <= 5 MB received per rank and step."""
    import ctypes

    from paper_0809_1810_b200 import _lib

    lib = _lib.load()
    lv, p, world = 9, 20, 8
    bounds = D.row_bounds(lv, world)
    kc = D.coarse_cut(lv, bounds)
    pyramid = sum(4**k for k in range(2, lv + 1)) * (p + 1) * 16
    for r, (lo, hi) in enumerate(bounds):
        cb, hb = ctypes.c_size_t(), ctypes.c_size_t()
        assert lib.vfmm_shard_exchange_size(2_000_000, lv, p, lo, hi, kc, ctypes.byref(cb), ctypes.byref(hb)) == 0
        below, above = D.neighbours(bounds, r)
        recv = world * cb.value + hb.value * ((below is not None) + (above is not None))
        assert recv <= 5_000_000, recv
        assert recv < pyramid / 50
    # a level above kc that is not fine for the strip is rejected
    cb, hb = ctypes.c_size_t(), ctypes.c_size_t()
    lo, hi = bounds[1]
    assert lib.vfmm_shard_exchange_size(1000, lv, p, lo, hi, kc - 1, ctypes.byref(cb), ctypes.byref(hb)) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4, 8, 16])
def test_gpu_shard_kernels_match_single_gpu(world):
    from paper_0809_1810_b200 import workloads as W

    w = W.config1()
    dev = torch.device("cuda", 0)
    t = [torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma)]
    cfg = vf.FmmConfig(w.levels, w.order, G)
    dom = vf.Domain(*W.DOMAIN)
    ref, st = vf.evaluate_arrays(*t, cfg, dom)
    vel, m2l, near = D.evaluate_emulated(*t, cfg, dom, world)
    assert m2l == st.m2l_count and near == st.near_pair_count
    assert float((vel - ref).abs().max() / ref.abs().max()) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 8])
def test_gpu_shard_kernels_config2_full_size(world):
    """Config 2 (N = 2^20, l = 7, p = 17) on W logical ranks vs the single-GPU evaluate."""
    from paper_0809_1810_b200 import workloads as W

    w = W.config2()
    dev = torch.device("cuda", 0)
    t = [torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma)]
    cfg = vf.FmmConfig(w.levels, w.order, G)
    dom = vf.Domain(*W.DOMAIN)
    ref, st = vf.evaluate_arrays(*t, cfg, dom)
    vel, m2l, near = D.evaluate_emulated(*t, cfg, dom, world)
    assert m2l == st.m2l_count and near == st.near_pair_count
    assert float((vel - ref).abs().max() / ref.abs().max()) <= 1e-12


@pytest.mark.gpu
def test_nccl_world1_sharded_path_matches_evaluate():
    """The real NCCL orchestration (all_to_all_single, all_reduce on device
    tensors) end to end on one GPU."""
    from paper_0809_1810_b200 import workloads as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        w = W.config1()
        t = [torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma)]
        cfg = vf.FmmConfig(w.levels, w.order, G)
        dom = vf.Domain(*W.DOMAIN)
        ref, st = vf.evaluate_arrays(*t, cfg, dom)
        ids = torch.arange(w.n, device=dev)
        own, vel, sst = D.evaluate_sharded(*t, ids, cfg, dom)
        full = D.gather_velocities(own, vel, w.n)
        assert sst.m2l_count == st.m2l_count and sst.near_pair_count == st.near_pair_count
        assert float((full.t() - ref).abs().max() / ref.abs().max()) <= 1e-12
    finally:
        dist.destroy_process_group()
