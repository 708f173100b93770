"""Where the end-to-end (host buffers) time of a C5 sort goes: pinned H2D of
the arena, the sort itself, allocation + first touch of the output arrays,
and the whole s5_sort(sset) call."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1403_2056_b200 import corpora, ssss  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402
from paper_1403_2056_b200.strset import StringSet  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
n = int((1 << 28) * scale)
arena, alen, h = corpora.gen_nodup_device(n)
pin = torch.empty(alen, dtype=torch.uint8, pin_memory=True)
pin.copy_(arena[:alen])
hh = torch.empty(n, dtype=torch.int64, pin_memory=True)
hh.copy_(h)
del arena, h
torch.cuda.empty_cache()
dev = torch.empty(alen + 64, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev[:alen].copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
print(f"H2D pinned {alen / 1e9:.2f} GB: {1e3 * (t1 - t0):.1f} ms = {alen / (t1 - t0) / 1e9:.1f} GB/s")
out = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(2):
    t0 = time.perf_counter()
    o = np.empty(n, dtype=np.int64)
    o2 = np.empty(n, dtype=np.int64)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    o[:] = 0
    o2[:] = 0
    t2 = time.perf_counter()
print(f"np.empty x2 {2 * 8 * n / 1e9:.1f} GB: alloc {1e3 * (t1 - t0):.1f} ms, first touch {1e3 * (t2 - t1):.1f} ms")
ot = torch.from_numpy(o)
t0 = time.perf_counter()
ot.copy_(out)
t1 = time.perf_counter()
print(f"D2H 8n into touched pageable: {1e3 * (t1 - t0):.1f} ms = {8 * n / (t1 - t0) / 1e9:.1f} GB/s")
del dev, out
torch.cuda.empty_cache()
sset = StringSet(pin.numpy(), hh.numpy())
for i in range(3):
    t0 = time.perf_counter()
    r = ssss.s5_sort(sset, want_lcps=True)
    t1 = time.perf_counter()
    print(f"s5_sort(sset) e2e #{i}: {1e3 * (t1 - t0):.1f} ms")
