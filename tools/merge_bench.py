"""Time the GPU K-way LCP merge of K sorted parts of a config (s5g_kway_merge)."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1403_2056_b200 import _lib, corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_dna")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--K", type=int, default=8)
a = ap.parse_args()
buf, hnd = corpora.CONFIGS[a.config](a.scale)
n = len(hnd)
ds = D.upload(buf, hnd)
cuts = np.linspace(0, n, a.K + 1).astype(np.int64)
run_h = torch.empty(n, dtype=torch.int64, device="cuda")
run_l = torch.empty_like(run_h)
run_c = torch.empty(n, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for j in range(a.K):
    sub = D.DeviceStrings(ds.arena, ds.arena_len, ds.handles[cuts[j]:cuts[j + 1]])
    h, l, c = D.sort(sub, want_lcps=True, want_dchar=True)
    run_h[cuts[j]:cuts[j + 1]] = h
    run_l[cuts[j]:cuts[j + 1]] = l
    run_c[cuts[j]:cuts[j + 1]] = c
e1.record()
torch.cuda.synchronize()
t_sort = e0.elapsed_time(e1)
full_h, full_l, _ = D.sort(ds, want_lcps=True)
for cached in (False, True):
    times = []
    for rep in range(4):
        st = _lib.Stats()
        e0.record()
        oh, ol = D.kway_merge(ds, cuts, run_h, run_l, run_c if cached else None, 0, st)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ok = torch.equal(oh, full_h) and torch.equal(ol[1:], full_l[1:])
    t = min(times[1:])
    print(f"{a.config} n={n} K={a.K} cached={cached}: merge {t:.3f} ms = {n / t / 1e6:.2f} G strings/s, "
          f"word loads {st.word_fetches / n:.2f}/string, equal to one-shot sort: {ok}")
print(f"sorting the {a.K} parts: {t_sort:.3f} ms")
