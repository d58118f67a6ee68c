"""CPU-side checks: the C-ABI library loads and exports every symbol of
include/vfmm.h, its host-only entry points behave, and the Python mirror of the
reference API validates like the reference (engine.py:49-55, 346-347) and
fails loudly without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

from paper_0809_1810_b200 import _lib
import paper_0809_1810_b200 as vf

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "vfmm.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int64_t|int|const char\*)\s+(vfmm_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert set(names) == set(_lib.EXPORTED_SYMBOLS)
    for name in names:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.vfmm_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_workspace_size_and_layout():
    for n, lv, p in [(1, 2, 0), (4096, 3, 10), (65536, 5, 12), (1 << 20, 7, 17)]:
        size = _lib.workspace_size(n, lv, p)
        lay = _lib.layout(n, lv, p)
        assert lay.total == size
        offs = [lay.perm, lay.leaf_key, lay.leaf_starts, lay.sources, lay.near_uv, lay.mult, lay.loc, lay.counts]
        assert all(0 < o < size for o in offs)
        cells = sum(4**k for k in range(2, lv + 1))
        assert size >= cells * (p + 1) * 16 * 2 + n * (32 + 16 + 16)


def test_invalid_arguments_rejected_without_touching_the_gpu():
    lib = _lib.load()
    sz = ctypes.c_size_t()
    assert lib.vfmm_workspace_size(0, 3, 4, ctypes.byref(sz)) == _lib.VFMM_EINVAL
    assert lib.vfmm_workspace_size(10, 1, 4, ctypes.byref(sz)) == _lib.VFMM_EINVAL
    assert lib.vfmm_workspace_size(10, 3, 61, ctypes.byref(sz)) == _lib.VFMM_EINVAL
    assert lib.vfmm_workspace_size(10, 3, -1, ctypes.byref(sz)) == _lib.VFMM_EINVAL
    st = _lib.VfmmStats()
    # NULL inputs -> EINVAL before any CUDA call
    rc = lib.vfmm_evaluate(None, None, None, None, 10, 0.0, 0.0, 1.0, 3, 4, 0, None, None, None, 0,
                           _lib.FLAG_STATS, ctypes.byref(st), None)
    assert rc == _lib.VFMM_EINVAL
    # n >= 2^30 (32-bit sorted indices): rejected by the size query AND by the
    # evaluate entry points before any layout / CUDA work (fake non-null pointers)
    big = 1 << 30
    assert lib.vfmm_workspace_size(big, 3, 4, ctypes.byref(sz)) == _lib.VFMM_EINVAL
    assert lib.vfmm_workspace_size(big - 1, 3, 4, ctypes.byref(sz)) == _lib.VFMM_OK
    fake = ctypes.c_void_p(256)
    for fn in (lib.vfmm_evaluate, lib.vfmm_evaluate_host):
        rc = fn(fake, fake, fake, fake, big, 0.0, 0.0, 1.0, 3, 4, 1, fake, fake, fake, 1 << 40,
                _lib.FLAG_STATS, ctypes.byref(st), None)
        assert rc == _lib.VFMM_EINVAL
    rc = lib.vfmm_evaluate_shard(fake, fake, fake, fake, big, 0.0, 0.0, 1.0, 3, 4, 1, 0, 8, fake, fake,
                                 fake, 1 << 40, _lib.FLAG_PHASE_UP, ctypes.byref(st), None)
    assert rc == _lib.VFMM_EINVAL
    nbad = ctypes.c_int64()
    assert lib.vfmm_evaluate_at(fake, fake, 4, big, 0.0, 0.0, 1.0, 3, 4, 1, fake, fake, fake,
                                ctypes.byref(nbad), None) == _lib.VFMM_EINVAL


def test_config_validation_matches_reference():
    with pytest.raises(ValueError, match="levels must be >= 2"):
        vf.FmmConfig(levels=1, order=4).validate()
    with pytest.raises(ValueError, match="order must be >= 0"):
        vf.FmmConfig(levels=3, order=-1).validate()
    with pytest.raises(ValueError, match="exceeds cap 60"):
        vf.FmmConfig(levels=3, order=61).validate()
    vf.FmmConfig(levels=2, order=0).validate()
    with pytest.raises(ValueError):
        vf.evaluate([], vf.FmmConfig(3, 4))


def test_to_arrays_and_enclosing_domain():
    parts = [vf.Particle(0.5, 2.0, 1.0, 0.1), vf.Particle(-1.0, 0.5, -2.0, 0.2)]
    x, y, g, s = vf.to_arrays(parts)
    assert x.tolist() == [0.5, -1.0] and y.tolist() == [2.0, 0.5]
    assert g.tolist() == [1.0, -2.0] and s.tolist() == [0.1, 0.2]
    d = vf.enclosing_domain(parts)
    assert (d.xmin, d.ymin, d.side) == (-1.0, 0.5, 1.5)
    assert vf.enclosing_domain([vf.Particle(0.3, 0.3, 1.0, 0.1)]).side == 1.0


def test_to_arrays_accepts_ints_tuples_and_duck_typed_particles():
    """Integer fields, a tuple instead of a list and objects that only share the
    reference's field names (model.py:29-36, 125-137) all unpack to float64 arrays."""
    from types import SimpleNamespace

    parts = (vf.Particle(1, 2, 3, 1), SimpleNamespace(x=0.25, y=-0.5, gamma=np.float32(0.5), sigma=0.125))
    x, y, g, s = vf.to_arrays(parts)
    for a in (x, y, g, s):
        assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"] and a.shape == (2,)
    assert x.tolist() == [1.0, 0.25] and y.tolist() == [2.0, -0.5]
    assert g.tolist() == [3.0, 0.5] and s.tolist() == [1.0, 0.125]
    # None becomes NaN, as in numpy's own conversion the reference uses (the
    # evaluate then rejects the particle as outside the domain)
    assert np.isnan(vf.to_arrays([vf.Particle(0.0, None, 1.0, 0.1)])[1][0])


def test_grid_indices_floor_rule_and_clamp():
    dom = vf.Domain(0.0, 0.0, 1.0)
    ix, iy = vf.grid_indices(np.array([0.0, 0.5, 1.0, 0.24999999]), np.array([1.0, 0.25, 0.0, 0.75]), 4, dom)
    assert ix.tolist() == [0, 2, 3, 0] and iy.tolist() == [3, 1, 0, 3]


def test_kernel_kind_accepts_reference_values():
    from paper_0809_1810_b200.kernels import kernel_code
    assert kernel_code(vf.KernelKind.POINT_VORTEX) == 0
    assert kernel_code(vf.KernelKind.GAUSSIAN_BLOB) == 1
    assert kernel_code("gaussian_blob") == 1
    with pytest.raises(ValueError):
        kernel_code("nope")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_fails_loudly_without_cuda():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        vf.evaluate([vf.Particle(0.1, 0.1, 1.0, 0.01)], vf.FmmConfig(3, 4), vf.Domain(0, 0, 1))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        vf.velocity_direct([(0.0, 0.0)], [vf.Particle(0.1, 0.1, 1.0, 0.01)], vf.KernelKind.POINT_VORTEX)
