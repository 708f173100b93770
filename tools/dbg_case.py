import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, golden_io as G, paper_1403_2056_b200 as P
c = G.case("deep_prefix_1500")
buf = c["buffer_bytes"]
def sb(h): 
    e = buf.index(b"\0", h); return buf[h:e]
for tm in [1000, 600, 300]:
    s = P.StringSet(buf, c["handles"])
    res = P.s5_sort(s, depth=0, want_lcps=True, t_medium=tm, seed=5)
    oh, ol = c["out_handles"], c["lcps"]
    bad = np.flatnonzero((res.set.handles != oh) | (res.lcps != ol))
    print("t_medium", tm, "mismatches", len(bad))
    if len(bad):
        i = bad[0]
        for j in range(max(0, i-3), min(len(oh), i+4)):
            print(j, res.set.handles[j], oh[j], res.lcps[j], ol[j], sb(int(res.set.handles[j]))[24:], sb(int(oh[j]))[24:])
