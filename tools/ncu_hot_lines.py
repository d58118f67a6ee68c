"""Hot source lines (warp-stall samples, executed instructions) of one kernel
in an ncu report:  ncu_hot_lines.py <report> [n_lines] [kernel-regex]"""
import collections
import csv
import subprocess
import sys

cmd = ["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3], "-c", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
his = [i for i, x in enumerate(r) if x and x[0] == "Line No"]
hi = his[0]
h = r[hi]
ci = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


agg = collections.OrderedDict()
cur = None
end = his[1] if len(his) > 1 else len(r)
for x in r[hi + 1:end]:
    if len(x) <= si:
        continue
    if x[0].strip():
        cur = (x[0], x[1][:90])
        agg.setdefault(cur, [0.0, 0.0])
    if cur:
        agg[cur][0] += f(x[ci])
        agg[cur][1] += f(x[si])
tot = sum(v[0] for v in agg.values()) or 1
stot = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{k[0]:>5} inst {v[0]/tot*100:5.1f}% stall {v[1]/stot*100:5.1f}%  {k[1]}")
