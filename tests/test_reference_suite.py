"""Harness integration: the reference's OWN test
suite -- ``test_engine.py`` (TestEvaluate, TestBoundBudgets, TestEvaluateAt,
TestFullBudgetRun) and ``test_acceptance.py`` (criteria 1-9, including the
``run_sweep`` study with resume and the ``timing_study`` crossover) -- run with
``vortexfmm.engine.evaluate`` / ``evaluate_at`` and ``vortexfmm.harness.evaluate``
swapped for the GPU path (tests/ref_plugin/vfmm_dropin.py, the monkeypatch of
INTEGRATION.md).  The reference is the unmodified package installed by
tools/install_reference.sh into the git-ignored baseline/_ref/ (skipped when
absent); nothing of it is tracked in this repository."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "reference_tests")

pytestmark = pytest.mark.gpu

SELECT = [
    "test_engine.py::TestEvaluate",
    "test_engine.py::TestBoundBudgets",
    "test_engine.py::TestEvaluateAt",
    "test_engine.py::TestFullBudgetRun",
    "test_acceptance.py",
]


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference not installed (tools/install_reference.sh)")
def test_reference_suite_through_the_gpu_evaluate(tmp_path):
    report = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REF_TESTS, os.path.join(REPO, "tests", "ref_plugin"), REPO])
    env["VFMM_DROPIN_REPORT"] = str(report)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    ini = tmp_path / "pytest.ini"
    ini.write_text("[pytest]\n")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "vfmm_dropin", "-p", "no:cacheprovider",
           "-c", str(ini), "--rootdir", REF_TESTS] + [os.path.join(REF_TESTS, s) for s in SELECT]
    cfg = os.path.join(REF_TESTS, "study.cfg")  # criterion 7 reads ./study.cfg (the package root)
    if os.path.exists(cfg):
        (tmp_path / "study.cfg").write_text(open(cfg).read())
    out = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1500)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    print(tail)
    assert out.returncode == 0, tail
    calls = json.loads(report.read_text())
    # every evaluate of these tests went through the CUDA library
    assert calls["evaluate"] > 1000 and calls["evaluate_at"] >= 3, calls
    assert " passed" in out.stdout and " failed" not in out.stdout
