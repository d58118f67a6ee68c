"""Config-4 error study: FMM vs the O(N^2) direct sum with spatial error maps.

BASELINE.json configs[4] / SURVEY.md §8f-1: lattice Lamb-Oseen particles with
N in {2^12 .. 2^20}, l in 3..8, p in {5, 10, 15, 20, 25}; every FMM run is
compared with the regularised direct sum at every particle and binned into a
g x g error map (errors.compare / errors.spatial_map, reference
errors.py:46-120; the harness pattern of harness.py:211-267).  Both the FMM
and the direct sum run on the GPU; the report and the map are O(N) host work.

    python -m paper_0809_1810_b200.errorstudy --out study.csv --maps maps/
"""

from __future__ import annotations

import argparse
import csv
import os
import time
import warnings

import numpy as np
import torch

from . import errors, workloads
from .engine import FmmConfig, evaluate_arrays
from .kernels import KernelKind, velocity_direct_arrays
from .model import Domain

# the reference's sweep schema (harness.SWEEP_HEADER, harness.py:44-47)
HEADER = ["n", "l", "p", "seed", "distribution", "kernel", "max_abs", "max_rel", "rms_rel",
          "bound_violations", "sampled", "t_fmm_ms", "t_direct_ms", "m2l_count", "near_pair_count",
          "generator_id"]


def csv_row(n, levels, order, rep, violations, t_fmm_ms, t_direct_ms, st) -> list[str]:
    """One sweep row in the reference's formatting (harness.CaseResult.csv_row, harness.py:186-208)."""
    def g(v):
        return "NA" if v != v else format(v, ".10g")

    return [str(n), str(levels), str(order), "0", "lamb_oseen_lattice", "gaussian", g(rep.max_abs),
            g(rep.max_rel), g(rep.rms_rel), str(violations), "0", format(t_fmm_ms, ".3f"),
            format(t_direct_ms, ".3f"), str(st.m2l_count), str(st.near_pair_count), "lattice"]


_DIRECT_CACHE: dict = {}


def run_case(m: int, levels: int, order: int, grid: int = 8, device=None, budgets: bool = True,
             cache: bool = True):
    """One study case on the GPU; returns (report, map, stats, t_direct_ms).

    The particle set depends on the lattice size only, so the O(N^2) direct
    sum is computed once per (m, device) and reused for every (l, p) of the
    sweep (``cache=False`` recomputes it); the reported direct time is the
    measured time of that one sum."""
    w = workloads.config4(m, levels, order)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    dom = Domain(*workloads.DOMAIN)
    cols = [torch.from_numpy(a).to(dev) for a in (w.x, w.y, w.gamma, w.sigma)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # many (N, l) pairs violate the sigma guard by design
        vel, st = evaluate_arrays(*cols, FmmConfig(levels, order, KernelKind.GAUSSIAN_BLOB), dom)
    key = (m, str(dev))
    if cache and key in _DIRECT_CACHE:
        direct, t_direct = _DIRECT_CACHE[key]
    else:
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        u, v = velocity_direct_arrays(cols[0], cols[1], *cols, KernelKind.GAUSSIAN_BLOB)
        torch.cuda.synchronize(dev)
        t_direct = (time.perf_counter() - t0) * 1e3
        direct = torch.stack((u, v), dim=1).cpu().numpy()
        if cache:
            _DIRECT_CACHE[key] = (direct, t_direct)
    pos = np.stack((w.x, w.y), axis=1)
    bud = errors.bound_budgets(w.x, w.y, w.gamma, levels, order, dom) if budgets else None
    rep = errors.compare(vel.cpu().numpy().T, direct, pos, bud)
    return rep, errors.spatial_map(rep, dom, grid), st, t_direct


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--out", default="error_study.csv")
    ap.add_argument("--maps", default=None, help="directory for per-run error-map CSVs")
    ap.add_argument("--grid", type=int, default=8)
    ap.add_argument("--max-m", type=int, default=1024)
    args = ap.parse_args(argv)
    if args.maps:
        os.makedirs(args.maps, exist_ok=True)
    with open(args.out, "w", newline="") as fh:
        wr = csv.writer(fh, lineterminator="\n")
        wr.writerow(HEADER)
        for m, lv, p in workloads.CONFIG4_GRID:
            if m > args.max_m:
                continue
            rep, emap, st, t_dir = run_case(m, lv, p, args.grid)
            viol = len(errors.bound_check(rep)) if rep.bound_budget is not None else -1
            wr.writerow(csv_row(m * m, lv, p, rep, viol, st.t_total * 1e3, t_dir, st))
            fh.flush()
            if args.maps:
                errors.write_error_map_csv(emap, os.path.join(args.maps, f"map_n{m * m}_l{lv}_p{p}.csv"))


if __name__ == "__main__":
    main()
