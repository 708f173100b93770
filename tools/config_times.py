"""Median device time of the full sort (with LCPs) per config: 2 warm-up
sorts, then --reps timed ones (CUDA events on the current stream)."""
import argparse
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1_random,c2_dna,c3_urls,c4_suffixes,c5_nodup")
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--v", type=int, default=8191, help="splitter cap (tuning only)")
ap.add_argument("--t-medium", type=int, default=1 << 20,
                help="segments below it go to the finishers (tuning only; the library caps it at 2049)")
a = ap.parse_args()
for spec in a.configs.split(","):
    name, _, sc = spec.partition(":")
    scale = float(sc) if sc else 1.0
    if name == "c5_nodup":  # generated in HBM
        arena, alen, hd = corpora.gen_nodup_device(int((1 << 28) * scale))
        ds, hnd = D.DeviceStrings(arena, alen, hd), hd
    else:
        buf, hnd = corpora.CONFIGS[name](scale)
        ds = D.upload(buf, hnd)
    ws = torch.empty(D.workspace_bytes(len(hnd), 1 << 20), dtype=torch.uint8, device="cuda")
    out = (torch.empty(len(hnd), dtype=torch.int64, device="cuda"),
           torch.empty(len(hnd), dtype=torch.int64, device="cuda"))
    for _ in range(2):
        D.sort(ds, want_lcps=True, out=out, workspace=ws, v=a.v, t_medium=a.t_medium)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.sort(ds, want_lcps=True, out=out, workspace=ws, v=a.v, t_medium=a.t_medium)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    med = statistics.median(ts)
    print(f"{name}:{scale:g} n={len(hnd)}: median {med:.3f} ms (min {min(ts):.3f}, max {max(ts):.3f}) "
          f"= {len(hnd) / med / 1e6:.2f} G strings/s", flush=True)
    del ds, ws, out
    torch.cuda.empty_cache()
