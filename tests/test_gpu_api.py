"""GPU checks of the C-ABI contract beyond numerics (include/vfmm.h "Threading"
and the PHASE_UP / PHASE_DOWN rule): concurrent host threads, mismatched
OVERLAP flags between the sharded phases, PHASE_DOWN without PHASE_UP, the
asynchronous host path's domain check (quadtree.py:191-198: the reference
always raises) and the caller's current device being left alone."""
import ctypes
import threading

import numpy as np
import pytest
import torch

import paper_0809_1810_b200 as vf
from paper_0809_1810_b200 import _lib
from paper_0809_1810_b200 import distributed as D
from paper_0809_1810_b200 import workloads as W

pytestmark = pytest.mark.gpu

G = vf.KernelKind.GAUSSIAN_BLOB
DOM = vf.Domain(*W.DOMAIN)


def _case(seed, n=20000):
    rng = np.random.default_rng(seed)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    return x, y, rng.standard_normal(n) * 1e-4, np.full(n, 0.01)


def test_concurrent_threads_get_their_own_results():
    cfg = vf.FmmConfig(5, 12, G)
    cases = [_case(s) for s in range(4)]
    serial = [vf.evaluate_arrays(*c, cfg, DOM)[0].cpu().numpy() for c in cases]
    got = [[] for _ in cases]
    errors = []

    def work(i):
        try:
            torch.cuda.set_device(0)
            for _ in range(4):
                vel, st = vf.evaluate_arrays(*cases[i], cfg, DOM, overlap=bool(i & 1))
                got[i].append((vel.cpu().numpy(), st.near_pair_count))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i, runs in enumerate(got):
        assert len(runs) == 4
        for vel, _ in runs:
            assert np.array_equal(vel, serial[i]), f"thread {i}: result differs from its serial run"


@pytest.mark.parametrize("up_flags,down_flags", [(0, _lib.FLAG_OVERLAP), (_lib.FLAG_OVERLAP, 0), (0, 0)])
def test_sharded_phases_with_mismatched_overlap_flags(up_flags, down_flags):
    w = W.config0()
    t = [torch.as_tensor(a, device="cuda") for a in (w.x, w.y, w.gamma, w.sigma)]
    cfg = vf.FmmConfig(w.levels, w.order, G)
    ref, st = vf.evaluate_arrays(*t, cfg, DOM)

    def factory():
        return D.CudaShardBackend(t[0].device, private_workspace=True, up_flags=up_flags,
                                  down_flags=down_flags)

    vel, m2l, near = D.evaluate_emulated(*t, cfg, DOM, 2, backend_factory=factory)
    err = float((vel - ref).abs().max() / ref.abs().max())
    assert err <= 1e-12
    assert (m2l, near) == (st.m2l_count, st.near_pair_count)


def test_phase_down_without_phase_up_is_rejected():
    w = W.config0()
    t = [torch.as_tensor(a, device="cuda") for a in (w.x, w.y, w.gamma, w.sigma)]
    ws = vf.Workspace(w.n, w.levels, w.order, t[0].device)
    u = torch.empty_like(t[0])
    v = torch.empty_like(t[0])
    lib = _lib.load()
    rc = lib.vfmm_evaluate_shard(*(a.data_ptr() for a in t), w.n, *W.DOMAIN, w.levels, w.order, 1, 0,
                                 2**w.levels, u.data_ptr(), v.data_ptr(), ws.ptr, ws.nbytes,
                                 _lib.FLAG_PHASE_DOWN, None, None)
    assert rc == _lib.VFMM_EINVAL


def test_async_host_path_raises_out_of_domain():
    w = W.config0()
    x = w.x.copy()
    x[17] = 1.5  # outside [-1, 1]
    cfg = vf.FmmConfig(w.levels, w.order, G)
    pipe = vf.HostPipeline(w.n, cfg, DOM, depth=2)
    with pytest.raises(vf.OutOfDomainError, match=r"first indices \[17\]"):
        pipe.submit(x, w.y, w.gamma, w.sigma).result()
    # the same slots keep working on valid input afterwards
    ok = pipe.submit(w.x, w.y, w.gamma, w.sigma).result()
    assert np.isfinite(ok.numpy()).all()


def test_current_device_left_alone():
    before = torch.cuda.current_device()
    w = W.config0()
    vf.evaluate_arrays(w.x, w.y, w.gamma, w.sigma, vf.FmmConfig(3, 10, G), DOM)
    vf.evaluate_host(w.x, w.y, w.gamma, w.sigma, vf.FmmConfig(3, 10, G), DOM, graph=True)
    assert torch.cuda.current_device() == before
    torch.cuda.synchronize()
    assert torch.cuda.current_device() == before
