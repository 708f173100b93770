"""Launch timeline of one profiled sort (gap analysis)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1403_2056_b200 import _lib, corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_dna")
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
if a.config == "c5_nodup":  # generated in HBM
    arena, alen, h = corpora.gen_nodup_device(int((1 << 28) * a.scale))
    ds = D.DeviceStrings(arena, alen, h)
else:
    buf, hnd = corpora.CONFIGS[a.config](a.scale)
    ds = D.upload(buf, hnd)
for _ in range(3):
    D.sort(ds, want_lcps=True)
torch.cuda.synchronize()
_lib.profile(enable=True, reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
D.sort(ds, want_lcps=True)
e1.record()
torch.cuda.synchronize()
_lib.profile(enable=False)
print(f"sort total (torch events): {e0.elapsed_time(e1):.3f} ms")
last = {0: 0.0, 1: 0.0, 2: 0.0, 3: 0.0}
for name, s, t0, t1 in _lib.timeline():
    gap = t0 - last[s]
    last[s] = t1
    print(f"{"  " * s}{name:18s} s{s} {t0:8.3f} {t1:8.3f}  dur {t1 - t0:7.3f}  gap {gap:7.3f}")
_lib.finisher_counters(reset=True)
D.sort(ds, want_lcps=True)
torch.cuda.synchronize()
for k, v in _lib.finisher_counters().items():
    print(k, v)
