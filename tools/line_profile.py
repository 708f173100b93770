"""Per-source-line instruction and stall-sample shares of one kernel, from an
`ncu --page source --csv --print-source sass` export, mapped to lines with
`nvdisasm -g` of the same shared object (run where the export was made).

usage: python tools/line_profile.py SASS.csv LIB.so KERNEL_SUBSTR [TOP]
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

csv_path, lib, want = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(csv_path)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["h"] = r
    elif cur is not None:
        cur["rows"].append(r)
blk = next(b for b in blocks if want in b["name"])
h = blk["h"]
d = [r for r in blk["rows"] if len(r) == len(h)]
ie, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cub = glob.glob(tmp + "/*.cubin")[0]
dis = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout.splitlines()
# mangled-name section whose instruction count matches the export
secs, name, cur_line, idx = {}, None, None, {}
for l in dis:
    m = re.match(r"\s*\.section\s+\.text\.(\S+),", l) or re.match(r"\.text\.(\S+):", l)
    if m:
        name = m.group(1).rstrip(":")
        secs.setdefault(name, {})
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,6})\*/", l)
    if m and name:
        secs[name][int(m.group(1), 16) // 16] = cur_line
cands = [n for n, s in secs.items() if len(s) == len(d)]
print(f"kernel {blk['name'][:80]}: {len(d)} sass; matching sections: {cands[:3]}")
m = secs[cands[0]] if cands else {}
agg = collections.defaultdict(lambda: [0.0, 0])
tot = sum(float(r[ie] or 0) for r in d) or 1
tots = sum(int(r[si]) for r in d) or 1
for i, r in enumerate(d):
    agg[m.get(i)][0] += float(r[ie] or 0)
    agg[m.get(i)][1] += int(r[si])
print(f"warp-inst {tot:.0f}, stall samples {tots}")
for k, (a, b) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"  {str(k):36s} inst {100 * a / tot:5.1f}%  stall {100 * b / tots:5.1f}%")
