"""Per-phase device time of one distributed_sort at world size 1 (torchrun):
which parts of the multi-GPU orchestration cost what (CUDA events around
each backend call)."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402
from paper_1403_2056_b200 import dist as Dist  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0625
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl")
n = int((1 << 28) * scale)
arena, alen, h = corpora.gen_nodup_device(n)
ds = D.DeviceStrings(arena, alen, h)
be = Dist.GpuBackend()
times = {}


def wrap(name, fn):
    def f(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        times[name] = times.get(name, 0.0) + 1e3 * (time.perf_counter() - t0)
        return r
    return f


for name in ("prepare", "sample", "partition", "group_by_dest", "global_index", "pack", "unpack",
             "local_sort", "take", "string_bytes"):
    setattr(be, name, wrap(name, getattr(be, name)))
Dist._all_gather_strings = wrap("all_gather_strings", Dist._all_gather_strings)
Dist._alltoallv = wrap("alltoallv", Dist._alltoallv)
shard = Dist.Shard(ds, h.cpu().numpy(), 0)
for it in range(3):
    times.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Dist.distributed_sort(shard, be, want_lcps=True)
    torch.cuda.synchronize()
    tot = 1e3 * (time.perf_counter() - t0)
print(f"total {tot:.2f} ms (n = {n})")
for k, v in sorted(times.items(), key=lambda x: -x[1]):
    print(f"  {k:20s} {v:8.2f} ms")
dist.destroy_process_group()
