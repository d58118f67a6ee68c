"""CPU check of ``bench.py --impl reference`` (the reference arm the driver runs
next to ours): on the small config 0 it must print ONE JSON line carrying the
contract's keys, say whether the unmodified reference (baseline/_ref) or the
numpy port ran, and agree between the two when both are available."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.isdir(os.path.join(REPO, "baseline", "_ref", "vortexfmm"))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "0",
                          "--steps", "1", "--warmup", "0", "--ref-workers", "2"],
                         capture_output=True, text=True, env=env, timeout=300, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1, out
    return json.loads(lines[0])


@pytest.mark.parametrize("arm", ["port"] + (["reference"] if HAVE_REF else []))
def test_reference_arm_line(arm):
    line = _run({"VFMM_REF_ARM": "port"} if arm == "port" else {})
    assert line["impl"] == "reference" and line["higher_is_better"] is True
    assert line["config"]["workload"] == "config0_lattice64" and line["config"]["same_config"] is True
    assert line["cpu_baseline"]["kind"] == arm and line["cpu_baseline"]["cores"] == 2
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["unit"] == "particle-evals/s" and line["steps"] == 1
