"""Error-map pipeline: report, g x g map, bound budgets.

CPU: the host implementation (paper_0809_1810_b200.errors) fed by the oracle
reproduces the reference's reports and maps on the golden config-4 cases;
GPU: the full pipeline (GPU FMM + GPU direct sum) matches them per bin to
1e-12 * max|v_direct| (absolute: high-p maps are round-off noise)."""
import numpy as np
import pytest

from _golden import GOLDEN
from oracle import fmm_oracle as O
from paper_0809_1810_b200 import errors, workloads as W
from paper_0809_1810_b200.model import Domain

ERR_CASES = [str(c) for c in GOLDEN["err_cases"]]
BOX = Domain(-1.0, -1.0, 2.0)


def _check(pre, rep, emap, budgets=None):
    vmax = float(GOLDEN[pre + "vmax_direct"])
    tol = 1e-12 * vmax
    s = GOLDEN[pre + "scalars"]
    assert abs(rep.max_abs - s[0]) <= tol and abs(rep.rms_abs - s[2]) <= tol
    assert np.array_equal(emap.counts, GOLDEN[pre + "map_counts"])
    for key, got in (("map_max", emap.max_err), ("map_mean", emap.mean_err)):
        ref = GOLDEN[pre + key]
        assert np.array_equal(np.isnan(got), np.isnan(ref))
        ok = ~np.isnan(ref)
        assert np.abs(got[ok] - ref[ok]).max() <= tol
    if budgets is not None:
        assert len(errors.bound_check(rep)) == int(GOLDEN[pre + "violations"])


@pytest.mark.parametrize("name", ERR_CASES)
def test_host_error_pipeline_on_oracle_matches_reference(name):
    pre = f"err/{name}/"
    m, lv, p = (int(v) for v in GOLDEN[pre + "cfg"])
    if m > 64:
        pytest.skip("oracle direct sum too slow for the CPU suite")
    w = W.config4(m, lv, p)
    vel, _ = O.evaluate(w.x, w.y, w.gamma, w.sigma, lv, p, True, W.DOMAIN)
    direct = O.direct(w.x, w.y, w.x, w.y, w.gamma, w.sigma, True)
    bud = errors.bound_budgets(w.x, w.y, w.gamma, lv, p, BOX)
    np.testing.assert_allclose(bud[::37], GOLDEN[pre + "budgets_sample"], rtol=1e-14, atol=0)
    rep = errors.compare(vel, direct, np.stack((w.x, w.y), axis=1), bud)
    _check(pre, rep, errors.spatial_map(rep, BOX, 8), bud)


def test_error_map_csv_na_tokens(tmp_path):
    rep = errors.compare(np.array([[1.0, 0.0], [0.0, 1.0]]), np.array([[1.0, 0.5], [0.0, 1.0]]),
                         np.array([[-0.9, -0.9], [-0.8, -0.9]]))
    emap = errors.spatial_map(rep, BOX, 2)
    path = tmp_path / "m.csv"
    errors.write_error_map_csv(emap, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "bin_ix,bin_iy,count,max_err,mean_err"
    assert lines[1].startswith("0,0,2,0.5,0.25") and lines[2] == "1,0,0,NA,NA"
    with pytest.raises(ValueError):
        errors.compare(np.zeros((0, 2)), np.zeros((0, 2)), np.zeros((0, 2)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ERR_CASES)
def test_gpu_error_pipeline_matches_reference_maps(name):
    from paper_0809_1810_b200 import errorstudy

    pre = f"err/{name}/"
    m, lv, p = (int(v) for v in GOLDEN[pre + "cfg"])
    rep, emap, st, _ = errorstudy.run_case(m, lv, p, grid=8)
    _check(pre, rep, emap, rep.bound_budget)
