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


@pytest.mark.parametrize("depth,compute_streams", [(2, 0), (3, 1), (5, 2), (6, 4)])
def test_host_pipeline_layouts_are_bitwise_equal(depth, compute_streams):
    """The three-stream pipeline (vfmm_evaluate_host_streams: copies on shared
    copy streams, graphs on a few compute streams) and the one-stream-per-slot
    layout return, for every batch of a sequence, exactly what a synchronous
    evaluate_host returns -- also on the first submissions of each slot (stream
    launches, then the graph capture, then replays)."""
    cfg = vf.FmmConfig(4, 11, G)
    cases = [_case(s) for s in (3, 4, 5)]
    want = [vf.evaluate_host(*c, cfg, DOM)[0].clone() for c in cases]
    pipe = vf.HostPipeline(20000, cfg, DOM, depth=depth, compute_streams=compute_streams)
    pinned = [[torch.from_numpy(a).pin_memory() for a in c] for c in cases]
    pend = []
    for k in range(4 * depth + 3):
        p = pipe.submit(*pinned[k % 3])
        pend.append((k % 3, p))
        if len(pend) >= depth:  # consume before the slot comes round again
            j, q = pend.pop(0)
            assert torch.equal(q.result(), want[j])
    for j, q in pend:
        assert torch.equal(q.result(), want[j])
        assert q.done()


def test_host_streams_entry_rejects_bad_arguments():
    lib = _lib.load()
    w = W.config0()
    cfg = vf.FmmConfig(w.levels, w.order, G)
    pipe = vf.HostPipeline(w.n, cfg, DOM, depth=1, compute_streams=1)
    ws, _, out = pipe.slots[0]
    h = [torch.from_numpy(a).pin_memory() for a in (w.x, w.y, w.gamma, w.sigma)]
    h2d, d2h = pipe.copy_streams
    cs = pipe.compute[0]

    def call(flags, a, b, c):
        return lib.vfmm_evaluate_host_streams(
            h[0].data_ptr(), h[1].data_ptr(), h[2].data_ptr(), h[3].data_ptr(), w.n, DOM.xmin, DOM.ymin,
            DOM.side, w.levels, w.order, _lib.KERNEL_GAUSSIAN, out.data_ptr(), None, ws.ptr, ws.nbytes,
            flags, a, b, c)

    ok = _lib.FLAG_UV_PAIRS | _lib.FLAG_OVERLAP
    assert call(ok | _lib.FLAG_STATS, cs.cuda_stream, h2d.cuda_stream, d2h.cuda_stream) == _lib.VFMM_EINVAL
    assert call(ok, cs.cuda_stream, None, d2h.cuda_stream) == _lib.VFMM_EINVAL
    assert call(ok, cs.cuda_stream, cs.cuda_stream, d2h.cuda_stream) == _lib.VFMM_EINVAL
    assert call(ok, cs.cuda_stream, h2d.cuda_stream, d2h.cuda_stream) == _lib.VFMM_OK
    torch.cuda.synchronize()
    want = vf.evaluate_host(w.x, w.y, w.gamma, w.sigma, cfg, DOM)[0]
    assert torch.equal(out, want)


def test_async_three_stream_path_raises_out_of_domain():
    w = W.config0()
    x = w.x.copy()
    x[23] = -1.25
    cfg = vf.FmmConfig(w.levels, w.order, G)
    pipe = vf.HostPipeline(w.n, cfg, DOM, depth=3, compute_streams=2)
    for _ in range(4):  # through the stream-launch, capture and replay calls of a slot
        assert np.isfinite(pipe.submit(w.x, w.y, w.gamma, w.sigma).result().numpy()).all()
    with pytest.raises(vf.OutOfDomainError, match=r"first indices \[23\]"):
        pipe.submit(x, w.y, w.gamma, w.sigma).result()
    assert np.isfinite(pipe.submit(w.x, w.y, w.gamma, w.sigma).result().numpy()).all()


def test_current_device_left_alone():
    before = torch.cuda.current_device()
    w = W.config0()
    vf.evaluate_arrays(w.x, w.y, w.gamma, w.sigma, vf.FmmConfig(3, 10, G), DOM)
    vf.evaluate_host(w.x, w.y, w.gamma, w.sigma, vf.FmmConfig(3, 10, G), DOM, graph=True)
    assert torch.cuda.current_device() == before
    torch.cuda.synchronize()
    assert torch.cuda.current_device() == before
