"""Sanitizer substitutes (compute-sanitizer is closed on this GPU pool, see
DESIGN.md): the CHECKED build of libvfmm.so (-DVFMM_CHECKED: every VCHECK
bounds / invariant check traps) runs every kernel path without a trap, and
the JITTERED build (-DVFMM_JITTER: each warp sleeps a pseudo-random time at
kernel entry and inside the work loops, reshuffling warp interleavings and the
atomic work-cursor order) gives results BITWISE identical to the plain build
-- a warp-synchronous race, a missing barrier or an order-dependent
reduction would show up as a difference.  Both builds come from
``make -C paper_0809_1810_b200/csrc variants`` (run by __graft_entry__.build)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(REPO, "build", "checked", "libvfmm.so")
JITTER = os.path.join(REPO, "build", "jitter", "libvfmm.so")


def _run(args, lib=None, timeout=900):
    env = dict(os.environ)
    if lib:
        env["VFMM_LIB"] = lib
    return subprocess.run([sys.executable] + args, cwd=REPO, env=env, capture_output=True, text=True,
                          timeout=timeout)


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build missing (make variants)")
def test_checked_build_runs_every_path_without_a_trap():
    r = _run([os.path.join("tools", "sanitize_cases.py")], CHECKED)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize cases done" in r.stdout


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build missing (make variants)")
def test_checked_build_lsd_sort_path():
    env_cmd = [os.path.join("tools", "sanitize_cases.py"), "config0", "graph", "shard"]
    env = dict(os.environ, VFMM_LIB=CHECKED, VFMM_SORT="lsd")
    r = subprocess.run([sys.executable] + env_cmd, cwd=REPO, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.skipif(not os.path.exists(JITTER), reason="jitter build missing (make variants)")
def test_jittered_build_is_bitwise_identical(tmp_path):
    plain, jit = tmp_path / "plain.npz", tmp_path / "jitter.npz"
    r = _run([os.path.join("tools", "dump_cases.py"), str(plain)])
    assert r.returncode == 0, r.stderr[-2000:]
    for rep in range(2):
        r = _run([os.path.join("tools", "dump_cases.py"), str(jit)], JITTER)
        assert r.returncode == 0, r.stderr[-2000:]
        a, b = np.load(plain), np.load(jit)
        assert sorted(a.files) == sorted(b.files)
        for k in a.files:
            assert np.array_equal(a[k], b[k]), f"{k} differs under jitter (run {rep})"
