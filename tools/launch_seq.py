import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]; col = {k: j for j, k in enumerate(h)}
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
seq=[]
for r in rows[start + 1:]:
    if len(r) < len(h) or r[col["Metric Name"]] != "gpu__time_duration.sum": continue
    name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "").replace("s5g::", "")
    ms = float(r[col["Metric Value"]].replace(",", "")) * scale[r[col["Metric Unit"]]]
    seq.append((name[:60], ms))
# print last third (3 iterations -> last one)
n=len(seq)//3
for nm,ms in seq[-n:]:
    if ms>0.05: print(f"{nm:60s} {ms:8.3f}")
print("total", sum(ms for _,ms in seq[-n:]))
