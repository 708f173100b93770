"""Dynamic code footprint and per-instruction stall reasons of each kernel in
an `ncu --page source --csv --print-source sass` export: how many SASS
instructions were executed at all (x 16 B = the instruction-cache footprint),
and which instructions carry the `no_instruction` (fetch) stall samples.
usage: python tools/code_footprint.py SASS.csv [FILTER [REASON,REASON...]]   (reasons: no_inst, long_sb, short_sb, barrier, wait ...)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["h"] = r
    elif cur is not None:
        cur["rows"].append(r)
seen = set()
for b in blocks:
    h = b.get("h")
    if not h or want not in b["name"]:
        continue
    sig = (b["name"], tuple(tuple(r[2:6]) for r in b["rows"][:64]))
    if sig in seen:  # ncu exports every launch twice
        continue
    seen.add(sig)
    ie = h.index("Instructions Executed")
    si = h.index("Warp Stall Sampling (All Samples)")
    d = [r for r in b["rows"] if len(r) == len(h)]
    ex = [i for i, r in enumerate(d) if float(r[ie] or 0) > 0]
    tot = sum(float(r[ie] or 0) for r in d)
    print(f"== {b['name'][:80]}  sass {len(d)} ({len(d) * 16 // 1024} KB)  executed {len(ex)} "
          f"({len(ex) * 16 // 1024} KB)  span {ex[0] if ex else 0}..{ex[-1] if ex else 0}")
    # footprint that covers 90 / 99 % of the executed instructions
    byc = sorted((float(r[ie] or 0) for r in d), reverse=True)
    acc, marks = 0.0, {}
    for k, c in enumerate(byc):
        acc += c
        for p in (0.5, 0.9, 0.99):
            if p not in marks and acc >= p * tot:
                marks[p] = k + 1
    print("   instructions covering 50/90/99 % of executed:", marks)
    stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_")]
    if stall_cols:
        tots = {h[i]: sum(float(r[i] or 0) for r in d) for i in stall_cols}
        alls = sum(tots.values()) or 1
        print("   stalls:", ", ".join(f"{k[6:]} {100 * v / alls:.1f}%" for k, v in
                                      sorted(tots.items(), key=lambda kv: -kv[1])[:8]))
        for reason in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["no_inst"]):
            col = "stall_" + reason
            if col not in h:
                continue
            ni = h.index(col)
            rt = tots[col] or 1
            top = sorted(((float(r[ni] or 0), i, r[1].strip()[:70]) for i, r in enumerate(d)), reverse=True)[:14]
            for v, i, t in top:
                print(f"     {reason} {v:7.0f} ({100 * v / rt:4.1f}%) @{i:6d} {t}")
