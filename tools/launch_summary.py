"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv): launches and serialized ms per kernel, and the sort's total (the
corpus generator's and torch's own kernels excluded).
usage: python tools/launch_summary.py LAUNCHES.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
col = {k: j for j, k in enumerate(h)}
agg = collections.OrderedDict()
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for r in rows[start + 1:]:
    if len(r) < len(h) or r[col["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "").replace("s5g::", "")
    ms = float(r[col["Metric Value"]].replace(",", "")) * scale[r[col["Metric Unit"]]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += ms
ours = {k: v for k, v in agg.items() if not re.search(r"gen_|cub::|at::", k)}
tot = sum(v[1] for v in ours.values())
for k, v in sorted(ours.items(), key=lambda x: -x[1][1]):
    print(f"{k[:40]:40s} {v[0]:4d} {v[1]:9.3f} ms {100 * v[1] / tot:5.1f} %")
print(f"{'sort total (serialized)':40s} {sum(v[0] for v in ours.values()):4d} {tot:9.3f} ms")
