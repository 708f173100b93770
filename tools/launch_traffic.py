"""Per-kernel time and DRAM traffic of one full-size sort from an ncu launch
list taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum (one pass, no replay: it runs at C5's full 31 GB where a
--set full replay cannot), written as the traffic JSON bench.py reads for
roofline.traffic, and printed as a table.
usage: python tools/launch_traffic.py LAUNCHES.csv OUT.json [label]"""
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
col = {k: j for j, k in enumerate(h)}
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
launch = collections.defaultdict(dict)
names = {}
for r in rows[start + 1:]:
    if len(r) < len(h):
        continue
    lid = r[col["ID"]]
    names[lid] = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "").replace("s5g::", "")
    v = float(r[col["Metric Value"]].replace(",", "")) * scale.get(r[col["Metric Unit"]], 1.0)
    launch[lid][r[col["Metric Name"]]] = v
kern = collections.OrderedDict()
for lid, m in launch.items():
    name = names[lid]
    if re.search(r"gen_|cub::|at::", name):
        continue
    e = kern.setdefault(name, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    e["launches"] += 1
    e["ms"] += m.get("gpu__time_duration.sum", 0.0)
    e["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
for e in kern.values():
    e["dram_bytes_per_launch"] = e["dram_bytes"] / e["launches"]
label = sys.argv[3] if len(sys.argv) > 3 else "one sort"
json.dump({"source": f"ncu launch list (time + DRAM bytes, one pass, --clock-control none), {label}",
           "kernels": kern}, open(sys.argv[2], "w"), indent=1)
tot = sum(e["ms"] for e in kern.values())
tb = sum(e["dram_bytes"] for e in kern.values())
print(f"{'kernel':28s} {'n':>4s} {'ms':>9s} {'share':>6s} {'DRAM GB':>8s} {'GB/s':>7s}")
for k, e in sorted(kern.items(), key=lambda x: -x[1]["ms"]):
    print(f"{k:28s} {e['launches']:4d} {e['ms']:9.3f} {100 * e['ms'] / tot:5.1f}% "
          f"{e['dram_bytes'] / 1e9:8.3f} {e['dram_bytes'] / 1e6 / max(e['ms'], 1e-9):7.0f}")
print(f"{'total (serialized)':28s} {sum(e['launches'] for e in kern.values()):4d} {tot:9.3f}        "
      f"{tb / 1e9:8.3f} {tb / 1e6 / tot:7.0f}")
