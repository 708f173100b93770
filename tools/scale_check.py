"""Sort a large config once on the GPU, certify it with the oracle (K11),
and print the time -- a size check beyond the test suite's scales."""
import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402  (the checker)
from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5_nodup")
ap.add_argument("--scale", type=float, default=0.25)
a = ap.parse_args()
t0 = time.time()
buf, hnd = corpora.CONFIGS[a.config](a.scale)
print(f"generated n={len(hnd)} N={len(buf) / 1e9:.2f} GB in {time.time() - t0:.1f} s", flush=True)
ds = D.upload(buf, hnd)
for _ in range(2):
    h, l, _ = D.sort(ds, want_lcps=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h, l, _ = D.sort(ds, want_lcps=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{a.config} scale {a.scale}: {ms:.2f} ms/sort = {len(hnd) / ms / 1e6:.2f} G strings/s, "
      f"peak mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
t0 = time.time()
status, bad = oracle.certify(buf, hnd, h.cpu().numpy(), l.cpu().numpy())
print(f"certificate: {oracle.CERT_STATUS[status]} (first bad {bad}) in {time.time() - t0:.1f} s")
