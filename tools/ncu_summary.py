"""Summarise ncu reports (one kernel launch each, --set full) as JSON:
time, FP64 pipe, issue, occupancy, DRAM/L2 traffic, and the top stall
reasons per issue.  Usage: ncu_summary.py out.json name=report.ncu-rep ..."""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
]
STALL = "smsp__average_warps_issue_stalled_"


def summarise_all(path):
    """One entry per profiled launch (keyed by kernel name, first launch wins)."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    res = {}
    for vals in rows[2:]:
        d = summarise_row(rows[0], rows[1], vals)
        name = d["kernel"].split("(")[0].replace("unnamed>::", "").replace("void ", "").strip()
        res.setdefault(name, d)
    return res


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return summarise_row(rows[0], rows[1], rows[2])


def summarise_row(head, units, vals):
    d = {k: [vals[head.index(k)], units[head.index(k)]] for k in KEYS if k in head}
    stalls = []
    for i, k in enumerate(head):
        if k.startswith(STALL) and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((k[len(STALL):-len("_per_issue_active.ratio")], float(vals[i])))
            except ValueError:
                pass
    d["top_stalls_per_issue"] = [[n, round(v, 2)] for n, v in sorted(stalls, key=lambda x: -x[1])[:5]]
    d["kernel"] = vals[head.index("Kernel Name")] if "Kernel Name" in head else ""
    return d


if __name__ == "__main__":
    res = {}
    for arg in sys.argv[2:]:
        if "=" in arg:  # name=report with one launch
            name, path = arg.split("=", 1)
            res[name] = summarise(path)
        else:  # report with several launches: one entry per kernel
            res.update(summarise_all(arg))
    with open(sys.argv[1], "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: [v["gpu__time_duration.sum"], v["top_stalls_per_issue"][:3]] for k, v in res.items()}))
