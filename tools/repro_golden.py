"""Run every golden case x parameter set through s5_sort (host entry) and
D.sort (device entry) and report the first failure (debug helper)."""
import sys
import traceback

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import golden_io as G  # noqa: E402
import paper_1403_2056_b200 as P  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402

KWS = [{}, {"t_medium": 16}, {"t_medium": 200, "variant": "equal"}, {"v": 7, "t_medium": 40},
       {"seed": 5, "t_medium": 1000}]
only = sys.argv[1] if len(sys.argv) > 1 else None
mode = sys.argv[2] if len(sys.argv) > 2 else "both"
fails = 0
for name in G.cases():
    if only and name != only:
        continue
    c = G.case(name)
    for kw in KWS:
        for entry in (("host", "device") if mode == "both" else (mode,)):
            try:
                if entry == "host":
                    s = P.StringSet(c["buffer_bytes"], c["handles"])
                    res = P.s5_sort(s, depth=c["depth"], want_lcps=True, want_dchar=True, **kw)
                    h, l = res.set.handles, res.lcps
                else:
                    ds = D.upload(c["buffer_bytes"], c["handles"])
                    hh, ll, _ = D.sort(ds, depth=c["depth"], want_lcps=True, **kw)
                    h, l = hh.cpu().numpy(), ll.cpu().numpy()
                ok = np.array_equal(h, c["out_handles"]) and np.array_equal(l, c["lcps"])
                if not ok:
                    fails += 1
                    print("MISMATCH", name, kw, entry, flush=True)
            except Exception:
                fails += 1
                print("ERROR", name, kw, entry, flush=True)
                traceback.print_exc()
                sys.exit(1)
print("done, failures:", fails)
