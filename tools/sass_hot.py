"""Top stall-sampled SASS windows per kernel from an `ncu --page source
--csv --print-source sass` export.  ncu exports one block per captured
launch; blocks of the same kernel are merged (printed once), optionally only
kernels whose name contains FILTER.
usage: python tools/sass_hot.py SASS.csv [FILTER]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["h"] = r
    elif cur is not None:
        cur["rows"].append(r)
want = sys.argv[2] if len(sys.argv) > 2 else ""
merged = {}
for b in blocks:
    if not b.get("h") or want not in b["name"]:
        continue
    m = merged.get(b["name"])
    if m is None or len(m["rows"]) != len(b["rows"]):
        merged.setdefault(b["name"], b)
        continue
    si = b["h"].index("Warp Stall Sampling (All Samples)")
    ie = b["h"].index("Instructions Executed")
    for r0, r1 in zip(m["rows"], b["rows"]):  # same SASS: add the counts
        if len(r0) == len(b["h"]) and len(r1) == len(b["h"]):
            r0[si] = str(int(r0[si]) + int(r1[si]))
            r0[ie] = str(float(r0[ie] or 0) + float(r1[ie] or 0))
for b in merged.values():
    h = b.get("h")
    si = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    d = [r for r in b["rows"] if len(r) == len(h)]
    tot = sum(int(r[si]) for r in d) or 1
    inst = sum(float(r[ie] or 0) for r in d)
    print(f"== {b['name'][:90]}  samples {tot}  warp-inst {inst:.0f}  sass {len(d)}")
    W = 32
    wins = []
    for k in range(0, len(d), W):
        sm = sum(int(r[si]) for r in d[k:k + W])
        ins = sum(float(r[ie] or 0) for r in d[k:k + W])
        top = max(d[k:k + W], key=lambda r: int(r[si]))
        wins.append((sm, ins, k, top[1].strip()[:60]))
    for sm, ins, k, t in sorted(wins, reverse=True)[:12]:
        print(f"  @{k:5d} samples {sm:6d} ({100 * sm / tot:4.1f}%) inst {100 * ins / max(inst, 1):4.1f}%  top: {t}")
