"""Drop-in ``parallel_s5`` (parallel.py:468-492) on GPUs.

In the reference, p is the number of forked CPU workers sharing one set.
Here the fully parallel step is the device-wide S^5 step (every CTA a
shard, bucket-major/CTA-minor offsets -- the interleaved prefix sum of
parallel.py:379-385), so one GPU already runs the reference's phased
structure.  ``p`` counts GPUs; within one process the set is sorted on the
current device.  Multi-GPU runs use one process per GPU
(``paper_1403_2056_b200.dist``: sample-sort partition + NCCL all-to-all).
"""

from __future__ import annotations

import numpy as np

from .ssss import T_MEDIUM, check_set, s5_sort
from .strset import LCP_UNDEF, SortedWithLcp, SortStats


def parallel_s5(sset, p=None, want_lcps: bool = False, want_dchar: bool = False, seed: int = 1,
                variant: str = "unroll", stats=None, t_medium: int = T_MEDIUM):
    """Sample sort on the GPU; content order matches the sequential sorter."""
    want = want_lcps or want_dchar
    return s5_sort(sset, want_lcps=want, want_dchar=want_dchar, variant=variant, seed=seed,
                   stats=stats, t_medium=t_medium)


def partitioned_merge_sort(sset, K: int = 4, p=None, use_cache: bool = True,
                           want_lcps: bool = False, seed: int = 1, stats=None, merge_stats=None,
                           t_medium: int = T_MEDIUM):
    """Sort K byte-balanced parts independently, then LCP-merge them
    (parallel.py:885-994) -- both phases on the GPU: each part through
    s5g_sort (handles, LCPs, distinguishing characters), then one
    s5g_kway_merge of the K runs (cached comparisons when use_cache).  The
    result is the stable content order, identical to parallel_s5's."""
    from . import _lib
    from . import device as D

    import torch

    n = len(sset.handles)
    merge_stats = merge_stats if merge_stats is not None else SortStats()
    if n == 0 or K <= 1:
        return parallel_s5(sset, p, want_lcps=want_lcps, seed=seed, stats=stats,
                           t_medium=t_medium)
    if K > 16:
        raise ValueError("at most 16 parts per merge")
    handles = np.ascontiguousarray(sset.handles, dtype=np.int64)
    check_set(sset.buffer, handles)
    ds = D.upload(sset.buffer, handles)
    # split characters into K contiguous, byte-balanced parts (whole strings)
    lens = D.lengths(ds).cpu().numpy() + 1
    cum = np.cumsum(lens)
    total = int(cum[-1])
    cuts = [0] + [int(np.searchsorted(cum, total * k / K)) for k in range(1, K)] + [n]
    parts = [(cuts[k], cuts[k + 1]) for k in range(K) if cuts[k] < cuts[k + 1]]
    dev = ds.handles.device
    run_h = torch.empty(n, dtype=torch.int64, device=dev)
    run_l = torch.empty(n, dtype=torch.int64, device=dev)
    run_c = torch.empty(n, dtype=torch.uint8, device=dev) if use_cache else None
    off = np.zeros(len(parts) + 1, dtype=np.int64)
    for j, (lo, hi) in enumerate(parts):
        sub = D.DeviceStrings(ds.arena, ds.arena_len, ds.handles[lo:hi])
        st = _lib.Stats()
        h, l, c = D.sort(sub, want_lcps=True, want_dchar=use_cache, seed=seed,
                         t_medium=t_medium, stats=st)
        run_h[lo:hi] = h
        run_l[lo:hi] = l
        if use_cache:
            run_c[lo:hi] = c
        off[j + 1] = hi
        if stats is not None:
            for f in _lib.STATS_FIELDS:
                setattr(stats, f, getattr(stats, f) + int(getattr(st, f)))
    mst = _lib.Stats()
    out_h, out_l = D.kway_merge(ds, off, run_h, run_l, run_c, 0, mst)
    for tgt in (merge_stats, stats):
        if tgt is not None:
            for f in _lib.STATS_FIELDS:
                setattr(tgt, f, getattr(tgt, f) + int(getattr(mst, f)))
    out = sset.with_handles(out_h.cpu().numpy())
    if not want_lcps:
        return out
    lcps = out_l.cpu().numpy()
    lcps[0] = LCP_UNDEF
    return SortedWithLcp(out, lcps, None, merge_stats)
