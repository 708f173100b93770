"""Drop-in ``parallel_s5`` (parallel.py:468-492) on GPUs.

In the reference, p is the number of forked CPU workers sharing one set
(p=None: os.cpu_count(), parallel.py:64-65).  Here p is the number of GPUs
(p=None: every visible device) and one process drives them all through the
library's multi-device entry (s5g_sort_multi): a sample-sort partition
with p-1 string splitters cuts the output order into p ranges, each device
sorts its range with the full S^5 (whose device-wide step is itself the
reference's phased step: every CTA a shard, bucket-major/CTA-minor
offsets), and the part-boundary LCPs are fixed on the host
(_boundary_lcps, parallel.py:447-455).  p larger than the visible device
count raises ValueError.  The multi-PROCESS form (one process per GPU,
NCCL all-to-all) is ``paper_1403_2056_b200.dist``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .ssss import T_MEDIUM, _accumulate, check_set, s5_sort
from .strset import LCP_UNDEF, SortedWithLcp, SortStats


def visible_devices() -> int:
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def parallel_s5(sset, p=None, want_lcps: bool = False, want_dchar: bool = False, seed: int = 1,
                variant: str = "unroll", stats=None, t_medium: int = T_MEDIUM, devices=None):
    """Sample sort on p GPUs; the output is the stable content order, identical
    to s5_sort's (and the reference's).  `devices` (tests): explicit device
    ordinals, repeats allowed, instead of 0 .. p-1."""
    from . import _lib
    from . import device as D

    if variant not in _lib.VARIANTS:
        raise ValueError(f"unknown classify variant: {variant}")
    ndev = visible_devices()
    if devices is None:
        if p is None:
            p = max(ndev, 1)
        if p < 1:
            raise ValueError("p must be at least 1")
        if p > ndev:
            raise ValueError(f"p = {p} exceeds the {ndev} visible CUDA device(s)")
        devices = list(range(p))
    devices = [int(d) for d in devices]
    want = want_lcps or want_dchar
    stats = stats if stats is not None else SortStats()
    handles = np.ascontiguousarray(sset.handles, dtype=np.int64)
    n = len(handles)
    if len(devices) == 1 or n == 0:
        if devices and n:
            import torch

            with torch.cuda.device(devices[0]):
                return s5_sort(sset, want_lcps=want, want_dchar=want_dchar, variant=variant,
                               seed=seed, stats=stats, t_medium=t_medium)
        return s5_sort(sset, want_lcps=want, want_dchar=want_dchar, variant=variant, seed=seed,
                       stats=stats, t_medium=t_medium)
    check_set(sset.buffer, handles)
    D._require_cuda()
    arr = sset.buffer if isinstance(sset.buffer, np.ndarray) else \
        np.frombuffer(sset.buffer, dtype=np.uint8)
    oh = np.empty(n, dtype=np.int64)
    ol = np.empty(n, dtype=np.int64) if want else None
    od = np.empty(n, dtype=np.uint8) if want_dchar else None
    ids = (C.c_int32 * len(devices))(*devices)
    st = _lib.Stats()
    a = _lib.MultiArgs()
    a.arena = arr.ctypes.data if arr.size else None
    a.arena_len = arr.size
    a.handles = handles.ctypes.data
    a.n = n
    a.depth = 0
    a.out_handles = oh.ctypes.data
    a.out_lcps = ol.ctypes.data if ol is not None else None
    a.out_dchar = od.ctypes.data if od is not None else None
    a.num_devices = len(devices)
    a.device_ids = ids
    a.variant = _lib.VARIANTS[variant]
    a.v = 8191
    a.seed = int(seed) & ((1 << 64) - 1)
    a.t_medium = int(t_medium)
    a.stats = C.pointer(st)
    _lib.check(_lib.lib().s5g_sort_multi(C.byref(a)))
    _accumulate(stats, st)
    out = sset.with_handles(oh)
    if not want:
        return out
    return SortedWithLcp(out, ol, od, stats)


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
    out_h, out_l = D.kway_merge_any(ds, off[: len(parts) + 1], run_h, run_l, run_c, 0, mst)
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
