"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Bar (BASELINE.json north_star): fp64 velocities
within 1e-12 of the reference FMM relative to max|v| (the reference's own
global normalisation, errors.py:64-73), exact m2l_count / near_pair_count, exact
tree structure, bitwise run-to-run determinism."""
import math
import os
import warnings

import numpy as np
import pytest
import torch

import paper_0809_1810_b200 as vf
from paper_0809_1810_b200 import workloads as W
from paper_0809_1810_b200.engine import Workspace
from _golden import CASES, DIRECT_CASES, GOLDEN, eval_case, enclosing
from oracle import fmm_oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-12  # north_star: within 1e-12 relative (summation-order differences only)
G = vf.KernelKind.GAUSSIAN_BLOB
PT = vf.KernelKind.POINT_VORTEX


def run(x, y, g, s, levels, order, gauss, domain, overlap=False):
    cfg = vf.FmmConfig(levels, order, G if gauss else PT)
    dom = vf.Domain(*domain) if domain is not None else None
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        vel, st = vf.evaluate_arrays(x, y, g, s, cfg, dom, overlap=overlap)
    return vel.cpu().numpy().T.copy(), st, rec


@pytest.mark.parametrize("name", CASES)
def test_evaluate_matches_reference_golden(name):
    c = eval_case(name)
    vel, st, rec = run(c["x"], c["y"], c["gamma"], c["sigma"], c["levels"], c["order"], c["gauss"],
                       c["domain"] or enclosing(c["x"], c["y"]))
    assert st.m2l_count == c["m2l_count"]
    assert st.near_pair_count == c["near_pair_count"]
    assert st.sigma_guard_ok == c["sigma_guard_ok"]
    if not c["sigma_guard_ok"]:
        assert any("core radius" in str(w.message) for w in rec)
    got = vel if c["sample"] is None else vel[c["sample"]]
    ref = c["vel"]
    if c["vmax"] == 0.0:
        assert np.all(got == 0.0)
    else:
        err = np.abs(got - ref).max() / c["vmax"]
        assert err <= REL_TOL, f"{name}: max rel err {err:.3e}"


@pytest.mark.parametrize("name", ["config0", "config1", "big_leaf_l3", "cluster_corner_l4", "boundary_edges"])
def test_tree_structure_exact(name):
    """Stable leaf permutation, leaf starts and per-level counts equal the oracle bit for bit."""
    c = eval_case(name)
    dom = c["domain"] or enclosing(c["x"], c["y"])
    run(c["x"], c["y"], c["gamma"], c["sigma"], c["levels"], c["order"], c["gauss"], dom)
    n, lv, p = c["x"].size, c["levels"], c["order"]
    ws = Workspace.get(n, lv, p, torch.device("cuda", torch.cuda.current_device()))
    tree = O.Tree(O.leaf_keys(c["x"], c["y"], lv, *dom), lv, *dom)
    perm = ws.view("perm", torch.int32, n).cpu().numpy()
    keys = ws.view("leaf_key", torch.int32, n).cpu().numpy()
    starts = ws.view("leaf_starts", torch.int32, 4**lv + 1).cpu().numpy()
    assert np.array_equal(perm, tree.order)
    assert np.array_equal(keys, tree.sorted_leaf)
    assert np.array_equal(starts, tree.leaf_starts)
    counts = ws.view("counts", torch.int32, sum(4**k for k in range(lv + 1))).cpu().numpy()
    off = 0
    for k in range(lv + 1):
        assert np.array_equal(counts[off: off + 4**k], tree.counts[k])
        off += 4**k


def _fuzz_case(seed):
    """Random (n, levels, distribution) across the build's mode boundaries: buckets with the
    scan fused into the pack (l <= 7, >= ~5 particles per leaf), buckets with the scan launch
    (l = 8), the scatter path (sparse leaves), a leaf above 128 (LSD fallback), tiny inputs."""
    rng = np.random.default_rng(1000 + seed)
    lv = int(rng.integers(2, 9))
    occ = [0.3, 2.0, 7.0, 30.0, 70.0][seed % 5]
    n = int(max(1, min(400_000, occ * 4**lv * rng.uniform(0.7, 1.3))))
    kind = seed % 4
    if kind == 0:  # uniform
        x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    elif kind == 1:  # clustered: some leaves far above the mean
        c = rng.uniform(-0.8, 0.8, (4, 2))
        w = rng.integers(0, 4, n)
        x = np.clip(c[w, 0] + 0.05 * rng.standard_normal(n), -1, 1)
        y = np.clip(c[w, 1] + 0.05 * rng.standard_normal(n), -1, 1)
    elif kind == 2:  # lattice, row-major (coherent order), with points on cell edges
        m = max(1, int(np.sqrt(n)))
        gx, gy = np.meshgrid(np.linspace(-1, 1, m), np.linspace(-1, 1, m))
        x, y = gx.ravel().copy(), gy.ravel().copy()
    else:  # uniform, a few duplicates and domain corners
        x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        x[: min(n, 4)] = [-1.0, 1.0, -1.0, 1.0][: min(n, 4)]
        y[: min(n, 4)] = [-1.0, -1.0, 1.0, 1.0][: min(n, 4)]
        if n > 10:
            x[5:10] = x[4]
            y[5:10] = y[4]
    n = x.size
    return x, y, rng.standard_normal(n) * 1e-3, np.full(n, 0.02), lv


@pytest.mark.parametrize("seed", range(20))
def test_tree_structure_exact_randomised(seed):
    """The build's outputs equal the oracle bit for bit and the velocities match it, across the
    mode boundaries of the counting path (see _fuzz_case)."""
    x, y, g, s, lv = _fuzz_case(seed)
    dom = (-1.0, -1.0, 2.0)
    order = 6
    vel, st, _ = run(x, y, g, s, lv, order, True, dom, overlap=bool(seed & 1))
    n = x.size
    ws = Workspace.get(n, lv, order, torch.device("cuda", torch.cuda.current_device()))
    tree = O.Tree(O.leaf_keys(x, y, lv, *dom), lv, *dom)
    assert np.array_equal(ws.view("perm", torch.int32, n).cpu().numpy(), tree.order)
    assert np.array_equal(ws.view("leaf_key", torch.int32, n).cpu().numpy(), tree.sorted_leaf)
    assert np.array_equal(ws.view("leaf_starts", torch.int32, 4**lv + 1).cpu().numpy(), tree.leaf_starts)
    counts = ws.view("counts", torch.int32, sum(4**k for k in range(lv + 1))).cpu().numpy()
    off = 0
    for k in range(lv + 1):
        assert np.array_equal(counts[off: off + 4**k], tree.counts[k])
        off += 4**k
    if n <= 60_000:  # the oracle's near field is O(n * 9 * leaf) python-side work
        ref, ost = O.evaluate(x, y, g, s, lv, order, True, dom)
        assert st.m2l_count == ost["m2l_count"] and st.near_pair_count == ost["near_pair_count"]
        vmax = np.abs(ref).max()
        assert vmax == 0.0 or np.abs(vel - ref).max() / vmax <= REL_TOL


def _unscale(ws, c, dom):
    """GPU multipoles/locals converted back to the reference convention."""
    n, lv, p = c["x"].size, c["levels"], c["order"]
    P = p + 1
    cells = sum(4**k for k in range(2, lv + 1))
    mult = ws.view("mult", torch.float64, cells * P * 2).cpu().numpy().reshape(-1, 2)
    loc = ws.view("loc", torch.float64, cells * P * 2).cpu().numpy().reshape(-1, 2)
    mult = (mult[:, 0] + 1j * mult[:, 1]).reshape(cells, P)
    loc = (loc[:, 0] + 1j * loc[:, 1]).reshape(cells, P)
    fact = np.array([math.factorial(k) for k in range(P)], dtype=np.float64)
    mult, loc = mult.reshape(-1), loc.reshape(-1)
    out_m, out_l, off = {}, {}, 0

    def cell_major(a, k):
        # planar [P][py][px][jy][jx] -> row-major cells [iy*m + ix][P]
        h = 2 ** (k - 1)
        return a.reshape(P, 2, 2, h, h).transpose(3, 1, 4, 2, 0).reshape(4**k, P)

    for k in range(2, lv + 1):
        r = dom[2] / 2**k
        kk = np.arange(P)
        out_m[k] = cell_major(mult[off: off + 4**k * P], k) * (r ** (kk + 1) * fact)[None, :]
        lk = cell_major(loc[off: off + 4**k * P], k)
        if k == lv:  # completed leaf locals live in the cell-major leaf array
            ll = ws.view("leaf_loc", torch.float64, 4**lv * P * 2).cpu().numpy().reshape(-1, 2)
            lk = (ll[:, 0] + 1j * ll[:, 1]).reshape(4**lv, P)
        out_l[k] = lk * (((-1.0) ** kk) / (fact * r**kk))[None, :]
        off += 4**k * P
    return out_m, out_l


@pytest.mark.parametrize("name", ["config1", "gauss_patch5000_l6_p4", "cluster_corner_l4"])
def test_expansions_match_oracle(name):
    """Every level's multipole and (completed) local coefficients vs the oracle."""
    c = eval_case(name)
    dom = c["domain"] or enclosing(c["x"], c["y"])
    run(c["x"], c["y"], c["gamma"], c["sigma"], c["levels"], c["order"], c["gauss"], dom)
    ws = Workspace.get(c["x"].size, c["levels"], c["order"], torch.device("cuda", torch.cuda.current_device()))
    _, st = O.evaluate(c["x"], c["y"], c["gamma"], c["sigma"], c["levels"], c["order"], c["gauss"], dom)
    gm, gl = _unscale(ws, c, dom)
    for k in range(2, c["levels"] + 1):
        om, ol = st["mult"][k], st["loc"][k]
        sm = np.abs(om).max(axis=0) + 1e-300
        sl = np.abs(ol).max(axis=0) + 1e-300
        assert (np.abs(gm[k] - om) / sm).max() <= 1e-12, f"mult level {k}"
        assert (np.abs(gl[k] - ol) / sl).max() <= 1e-11, f"loc level {k}"


def _symmetric_mode(c, n):
    """Mirror of p2p_symmetric (vfmm_internal.cuh): uniform sigma (or point kernel)
    and leaves of at most 128 particles select the symmetric near-field kernel."""
    if os.environ.get("VFMM_P2P_SYM") == "0":
        return False
    uniform = (not c["gauss"]) or np.all(c["sigma"] == c["sigma"][0])
    return uniform and np.bincount(O.leaf_keys(c["x"], c["y"], c["levels"], *(c["domain"] or enclosing(c["x"], c["y"])))).max() <= 128


def _near_from_slots(ws, c, n):
    """After an evaluate, slot 0 of near_uv holds each particle's complete near
    field (k_near_sum: own-leaf sums + backward reactions, or the three row
    partial sums), in sorted order."""
    return ws.view("near_uv", torch.float64, 2 * n).cpu().numpy().reshape(n, 2).copy()


@pytest.mark.parametrize("name", ["config0", "config1", "coincident", "big_leaf_l3", "point_kernel_l5"])
def test_near_field_matches_oracle(name):
    c = eval_case(name)
    dom = c["domain"] or enclosing(c["x"], c["y"])
    run(c["x"], c["y"], c["gamma"], c["sigma"], c["levels"], c["order"], c["gauss"], dom)
    n = c["x"].size
    ws = Workspace.get(n, c["levels"], c["order"], torch.device("cuda", torch.cuda.current_device()))
    near = _near_from_slots(ws, c, n)
    _, st = O.evaluate(c["x"], c["y"], c["gamma"], c["sigma"], c["levels"], c["order"], c["gauss"], dom)
    ref = st["near_sorted"]
    assert np.abs(near - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("overlap", [False, True])
def test_bitwise_determinism(overlap):
    w = W.config1()
    a, s1, _ = run(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN, overlap=overlap)
    b, s2, _ = run(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN, overlap=not overlap)
    assert np.array_equal(a, b)
    assert s1.m2l_count == s2.m2l_count and s1.near_pair_count == s2.near_pair_count


def test_generic_near_field_path_nonuniform_sigma():
    """Non-uniform core sizes select the generic (row-slice) near-field kernel."""
    w = W.config1()
    sig = w.sigma * (1.0 + 0.01 * np.cos(7 * w.x))
    vel, st, _ = run(w.x, w.y, w.gamma, sig, w.levels, w.order, True, W.DOMAIN)
    ref, ost = O.evaluate(w.x, w.y, w.gamma, sig, w.levels, w.order, True, W.DOMAIN)
    assert st.near_pair_count == ost["near_pair_count"] and st.m2l_count == ost["m2l_count"]
    assert np.abs(vel - ref).max() <= REL_TOL * np.abs(ref).max()


def test_drop_in_api_and_errors():
    parts = [vf.Particle(0.4, 0.6, 2.0, 0.01)]
    vel, st = vf.evaluate(parts, vf.FmmConfig(3, 6), vf.Domain(0.0, 0.0, 1.0))
    assert vel.shape == (1, 2) and np.all(vel == 0.0) and st.n == 1
    with pytest.raises(ValueError):
        vf.evaluate([], vf.FmmConfig(3, 4))
    bad = [vf.Particle(0.5, 0.5, 1.0, 0.01), vf.Particle(1.5, 0.5, 1.0, 0.01), vf.Particle(0.2, -0.1, 1.0, 0.01)]
    with pytest.raises(vf.OutOfDomainError, match=r"2 particle\(s\) outside domain .* first indices \[1, 2\]"):
        vf.evaluate(bad, vf.FmmConfig(3, 4), vf.Domain(0.0, 0.0, 1.0))
    with pytest.warns(UserWarning, match="core radius"):
        vf.evaluate([vf.Particle(0.5, 0.5, 1.0, 0.3), vf.Particle(0.6, 0.5, 1.0, 0.3)],
                    vf.FmmConfig(3, 4, G), vf.Domain(0.0, 0.0, 1.0))
    # stats contract of test_engine.py:272-285
    rng = np.random.default_rng(4)
    parts = [vf.Particle(float(a), float(b), float(c), 0.005) for a, b, c in rng.uniform(0, 1, (512, 3))]
    vel, st = vf.evaluate(parts, vf.FmmConfig(3, 6), vf.Domain(0.0, 0.0, 1.0))
    phases = st.t_build + st.t_upward + st.t_m2l + st.t_downward + st.t_eval + st.t_near
    assert st.t_total >= 0.95 * phases and st.t_total > 0
    assert st.m2l_count <= 27 * 4**3 and len(vel) == 512


@pytest.mark.parametrize("name", DIRECT_CASES)
def test_direct_matches_reference_golden(name):
    pre = f"direct/{name}/"
    tg = GOLDEN[pre + "targets"]
    if pre + "x" in GOLDEN:
        x, y, g, s = (GOLDEN[pre + k] for k in ("x", "y", "gamma", "sigma"))
    else:
        w = W.config0()
        x, y, g, s = w.x, w.y, w.gamma, w.sigma
    kind = G if int(GOLDEN[pre + "kind"]) else PT
    u, v = vf.velocity_direct_arrays(np.ascontiguousarray(tg[:, 0]), np.ascontiguousarray(tg[:, 1]), x, y, g, s, kind)
    got = np.stack((u.cpu().numpy(), v.cpu().numpy()), axis=1)
    ref = GOLDEN[pre + "vel"]
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_direct_reference_signature():
    parts = [vf.Particle(0.0, 0.0, 2 * math.pi, 1.0)]
    vel = vf.velocity_direct([(1.0, 0.0)], parts, G)
    assert vel[0, 0] == 0.0 and abs(vel[0, 1] - 0.3934693402873666) <= 1e-15
    vel = vf.velocity_direct([(1.0, 0.0)], [vf.Particle(0.0, 0.0, 2 * math.pi, 0.1)], PT)
    assert abs(vel[0, 1] - 1.0) <= 1e-15 and vel[0, 0] == 0.0


@pytest.mark.parametrize("gauss", [False, True])
def test_evaluate_at_matches_reference_golden(gauss):
    key = "at/grid_gauss/" if gauss else "at/grid/"
    x, y, g, s = (GOLDEN["at/grid/" + k] for k in ("x", "y", "gamma", "sigma"))
    tg = GOLDEN[key + "targets"]
    parts = [vf.Particle(*map(float, r)) for r in zip(x, y, g, s)]
    got = vf.evaluate_at(tg, parts, vf.FmmConfig(3, 20, G if gauss else PT), vf.Domain(0.0, 0.0, 1.0))
    ref = GOLDEN[key + "vel"]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    with pytest.raises(vf.OutOfDomainError):
        vf.evaluate_at([(1.5, 0.5)], parts, vf.FmmConfig(2, 4), vf.Domain(0.0, 0.0, 1.0))


# ---------------------------------------------------------------- full sizes
def _sampled_direct_check(w, vel, k=128, seed=0):
    """GPU direct sum at sampled targets == oracle direct (summation order only),
    and FMM close to the direct sum (truncation error only)."""
    sel = np.sort(np.random.default_rng(seed).choice(w.n, k, replace=False))
    u, v = vf.velocity_direct_arrays(w.x[sel], w.y[sel], w.x, w.y, w.gamma, w.sigma, G)
    gd = np.stack((u.cpu().numpy(), v.cpu().numpy()), axis=1)
    od = O.direct_blocked(w.x[sel], w.y[sel], w.x, w.y, w.gamma, w.sigma, True, block=1 << 16)
    vmax = np.abs(od).max()
    assert np.abs(gd - od).max() <= 1e-12 * vmax
    return np.abs(vel[sel] - gd).max() / vmax


def test_config2_full_size_properties():
    w = W.config2()
    vel, st, _ = run(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    assert st.m2l_count == 568_872 and st.near_pair_count == 596_656_128
    fmm_err = _sampled_direct_check(w, vel)
    assert fmm_err <= 1e-6
    # exact circulation scaling (every operation is linear in gamma)
    v2, _, _ = run(w.x, w.y, 2.0 * w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    assert np.array_equal(v2, 2.0 * vel)
    # linearity and permutation invariance to round-off
    g1 = w.gamma * np.cos(3 * w.x)
    va, _, _ = run(w.x, w.y, g1, w.sigma, w.levels, w.order, True, W.DOMAIN)
    vb, _, _ = run(w.x, w.y, w.gamma - g1, w.sigma, w.levels, w.order, True, W.DOMAIN)
    vmax = np.abs(vel).max()
    assert np.abs(va + vb - vel).max() <= 1e-13 * vmax
    perm = np.random.default_rng(5).permutation(w.n)
    vp, _, _ = run(w.x[perm], w.y[perm], w.gamma[perm], w.sigma[perm], w.levels, w.order, True, W.DOMAIN)
    assert np.abs(vp - vel[perm]).max() <= 1e-13 * vmax


@pytest.mark.slow
def test_config2_full_size_oracle_parity():
    w = W.config2()
    vel, st, _ = run(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    ov, ost = O.evaluate(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    assert st.m2l_count == ost["m2l_count"] and st.near_pair_count == ost["near_pair_count"]
    assert np.abs(vel - ov).max() <= REL_TOL * np.abs(ov).max()


@pytest.mark.slow
def test_config3_full_size_counts_and_sampled_direct():
    w = W.config3()
    vel, st, _ = run(w.x, w.y, w.gamma, w.sigma, w.levels, w.order, True, W.DOMAIN)
    assert st.m2l_count == 9_351_840 and st.near_pair_count == 9_638_451_922
    assert _sampled_direct_check(w, vel, k=24) <= 1e-6


@pytest.mark.parametrize("pinned", [True, False])
def test_host_buffer_entry_point_matches_device_path(pinned):
    """vfmm_evaluate_host (staged, overlapped copies) == vfmm_evaluate bit for bit."""
    w = W.config1()
    cfg = vf.FmmConfig(w.levels, w.order, G)
    dom = vf.Domain(*W.DOMAIN)
    ref, st = vf.evaluate_arrays(w.x, w.y, w.gamma, w.sigma, cfg, dom, overlap=True)
    arrs = (w.x, w.y, w.gamma, w.sigma)
    if pinned:
        arrs = tuple(torch.from_numpy(a).pin_memory() for a in arrs)
    got, st2 = vf.evaluate_host(*arrs, cfg, dom)
    assert torch.equal(got, ref.cpu().t())
    assert st2.m2l_count == st.m2l_count and st2.near_pair_count == st.near_pair_count


@pytest.mark.parametrize("levels,order,n", [(2, 60, 300), (4, 60, 2000), (10, 4, 10000), (11, 2, 3000)])
def test_extreme_orders_and_depths_match_oracle(levels, order, n):
    """ORDER_CAP (p = 60, depth-2 subtrees, long Hankel rows) and deep, mostly
    empty trees (up to 4^11 leaves) against the oracle."""
    rng = np.random.default_rng(levels * 100 + order)
    x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    g = rng.uniform(-1, 1, n)
    s = np.full(n, 1e-4)
    vel, st, _ = run(x, y, g, s, levels, order, True, (0.0, 0.0, 1.0))
    ref, ost = O.evaluate(x, y, g, s, levels, order, True, (0.0, 0.0, 1.0))
    assert st.m2l_count == ost["m2l_count"] and st.near_pair_count == ost["near_pair_count"]
    assert np.abs(vel - ref).max() <= REL_TOL * np.abs(ref).max()


@pytest.mark.gpu
def test_host_pipeline_matches_synchronous_call():
    """evaluate_host_async / HostPipeline (two calls in flight on their own
    workspaces and streams) give bitwise the results of evaluate_host."""
    w = W.config1()
    cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
    dom = vf.Domain(*W.DOMAIN)
    ref, st = vf.evaluate_host(w.x, w.y, w.gamma, w.sigma, cfg, dom)
    pipe = vf.HostPipeline(w.x.size, cfg, dom, depth=2)
    inputs = [(w.x, w.y, w.gamma * (1.0 + k), w.sigma) for k in range(4)]
    outs = []
    pend = [pipe.submit(*a) for a in inputs[:2]]
    for p, a in zip(pend, inputs[:2]):
        outs.append(p.result().clone())
    pend = [pipe.submit(*a) for a in inputs[2:]]
    last, st2 = pend[-1].result(with_stats=True)
    outs.append(pend[0].result().clone())
    outs.append(last.clone())
    for k, o in enumerate(outs):
        assert torch.equal(o, ref * (1.0 + k)) or np.abs((o - ref * (1.0 + k)).numpy()).max() <= 1e-13 * np.abs(ref.numpy()).max() * (1 + k)
    assert st2.near_pair_count == st.near_pair_count and st2.m2l_count == st.m2l_count


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["lattice", "random_order", "random_order_big_leaf", "mixed_sigma"])
def test_host_graph_path_matches_stream_launches(case):
    """VFMM_FLAG_GRAPH (cached CUDA graph of the device part) gives bitwise the
    stream-launched results: a coherent input (counting sort, symmetric P2P),
    a random-order one (counting sort below the LSD size threshold), a random
    one with a leaf of > 128 particles (LSD radix path chosen on the device
    inside the graph, generic P2P) and per-particle core sizes (generic P2P);
    replays reuse the cached graph with new input values, a different domain
    gets its own graph."""
    from paper_0809_1810_b200 import _lib

    rng = np.random.default_rng(7)
    if case == "lattice":
        w = W.config1()
        x, y, g, s = w.x, w.y, w.gamma, w.sigma
        levels, order = w.levels, w.order
    else:
        n = 20000
        x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        if case == "random_order_big_leaf":  # 300 particles in one leaf: the LSD path
            x[:300] = rng.uniform(0.50, 0.53, 300)
            y[:300] = rng.uniform(0.50, 0.53, 300)
        g = rng.standard_normal(n) * 1e-4
        s = np.full(n, 0.01) if case.startswith("random_order") else rng.uniform(0.005, 0.01, n)
        levels, order = 5, 12
    cfg = vf.FmmConfig(levels, order, vf.KernelKind.GAUSSIAN_BLOB)
    pinned = tuple(torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (x, y, g, s))
    for dom in (vf.Domain(*W.DOMAIN), vf.Domain(-1.5, -1.5, 3.0)):
        ref, st = vf.evaluate_host(*pinned, cfg, dom, graph=False)
        for scale in (1.0, -2.5):  # first call captures, the second replays the cached graph
            gin = pinned[2] * scale
            want = ref * scale if scale == 1.0 else vf.evaluate_host(pinned[0], pinned[1], gin, pinned[3],
                                                                      cfg, dom, graph=False)[0]
            before = _lib.load().vfmm_launch_count()
            got, st2 = vf.evaluate_host(pinned[0], pinned[1], gin, pinned[3], cfg, dom, graph=True)
            assert _lib.load().vfmm_launch_count() > before
            assert torch.equal(got, want)
            assert st2.m2l_count == st.m2l_count and st2.near_pair_count == st.near_pair_count
        pipe = vf.HostPipeline(x.size, cfg, dom, depth=2, graph=True)
        pend = [pipe.submit(*pinned) for _ in range(2)]
        for p in pend:
            assert torch.equal(p.result(), ref)


@pytest.mark.gpu
def test_programmatic_launch_off_is_bitwise_identical(tmp_path):
    """Programmatic dependent launch changes only when kernels are scheduled:
    an evaluate with the attribute disabled (VFMM_PDL=0, read at library load,
    so in a child process) gives bitwise the same velocities and counters."""
    import subprocess
    import sys

    w = W.config1()
    cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)
    vel, st = vf.evaluate_arrays(w.x, w.y, w.gamma, w.sigma, cfg, vf.Domain(*W.DOMAIN), overlap=True)
    out = tmp_path / "pdl_off.npy"
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_0809_1810_b200 as vf\n"
        "from paper_0809_1810_b200 import workloads as W\n"
        "w = W.config1(); cfg = vf.FmmConfig(w.levels, w.order, vf.KernelKind.GAUSSIAN_BLOB)\n"
        "v, st = vf.evaluate_arrays(w.x, w.y, w.gamma, w.sigma, cfg, vf.Domain(*W.DOMAIN), overlap=True)\n"
        "np.save(%r, np.concatenate([v.cpu().numpy().ravel(), [st.m2l_count, st.near_pair_count]]))\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), str(out))
    env = dict(os.environ, VFMM_PDL="0")
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=600)
    other = np.load(out)
    mine = np.concatenate([vel.cpu().numpy().ravel(), [st.m2l_count, st.near_pair_count]])
    assert np.array_equal(mine, other)


@pytest.mark.gpu
@pytest.mark.parametrize("env", ["VFMM_P2P_SPLIT=0", "VFMM_P2P_SPLIT=1", "VFMM_P2P_SPLIT_TAIL=1000",
                                 "VFMM_P2P_SPLIT_TAIL=0"])
def test_near_field_item_splits_agree(env, tmp_path):
    """The symmetric near field's work-item layouts -- one item per leaf, two
    per leaf, and a tail of two-item leaves (the TSPLIT kernel instance large
    random grids use, forced here on a 4,096-leaf grid) -- sum the same pairs
    in different orders: velocities agree to 1e-13 of max|v| (and with the
    oracle to 1e-12), counters exactly.  The layout is read from the
    environment at library load, so each runs in a child process."""
    import subprocess
    import sys

    rng = np.random.default_rng(11)
    n, levels, order = 40000, 6, 8
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    g = rng.normal(size=n)
    s = np.full(n, 0.004)
    src = tmp_path / "in.npz"
    np.savez(src, x=x, y=y, g=g, s=s)
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_0809_1810_b200 as vf\n"
        "d = np.load(%r); cfg = vf.FmmConfig(%d, %d, vf.KernelKind.GAUSSIAN_BLOB)\n"
        "v, st = vf.evaluate_arrays(d['x'], d['y'], d['g'], d['s'], cfg, vf.Domain(-1.0, -1.0, 2.0), overlap=True)\n"
        "np.save(sys.argv[1], np.concatenate([v.cpu().numpy().ravel(), [st.m2l_count, st.near_pair_count]]))\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), str(src), levels, order)
    outs = {}
    for tag, e in (("default", {}), ("variant", dict([env.split("=")]))):
        out = tmp_path / f"{tag}.npy"
        subprocess.run([sys.executable, "-c", code, str(out)], env=dict(os.environ, **e), check=True,
                       timeout=600)
        outs[tag] = np.load(out)
    a, b = outs["default"], outs["variant"]
    assert np.array_equal(a[-2:], b[-2:]), (a[-2:], b[-2:])
    va, vb = a[:-2], b[:-2]
    assert np.abs(va - vb).max() <= 1e-13 * np.abs(va).max()
    ref, _ = O.evaluate(x, y, g, s, levels, order, True, (-1.0, -1.0, 2.0))
    got = vb.reshape(2, n).T
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
