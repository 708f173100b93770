"""Exactly one sort (with LCPs) of a config, for ncu captures: no warm-up
sort, so every captured launch belongs to this one sort (ncu replays each
kernel itself; its times are cold-cache and serialised anyway)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_dna")
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
if a.config == "c5_nodup":  # generated in HBM (same bytes as the host generator)
    arena, alen, h = corpora.gen_nodup_device(int((1 << 28) * a.scale))
    ds, hnd = D.DeviceStrings(arena, alen, h), h
else:
    buf, hnd = corpora.CONFIGS[a.config](a.scale)
    ds = D.upload(buf, hnd)
out = D.sort(ds, want_lcps=True)
torch.cuda.synchronize()
print("one sort done", a.config, len(hnd))
