"""Drop-in GPU LCP merging (strsort.lcpmerge, lcpmerge.py:25-424).

``kway_lcp_merge`` / ``binary_lcp_merge`` keep the reference's signatures
and outputs -- the stable merge of sorted runs (ties to the earlier run) and
the LCP of every output string to its predecessor, ``out_lcps[0] =
LCP_UNDEF`` when the caller passes no output arrays, else ``shared`` -- and
run the merge in ``s5g_kway_merge`` (csrc/s5g_merge.cuh): candidate cuts by
LCP-bounded binary search, one LCP loser tree (lcp_compare /
lcp_compare_cached semantics) per job of ~32 strings, recomputed job
boundaries.  ``cached`` uses the runs' distinguishing characters.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as D
from .strset import LCP_UNDEF, SortStats


@dataclass
class LcpStream:
    """A sorted run with its LCP array and optional distinguishing chars
    (mirror of strsort.lcpmerge.LcpStream)."""

    sset: object
    handles: np.ndarray
    lcps: np.ndarray
    dchar: np.ndarray | None = None
    start: int = 0
    length: int | None = None

    def __post_init__(self):
        if self.length is None:
            self.length = len(self.handles) - self.start

    def slice(self, start: int, length: int) -> "LcpStream":
        return LcpStream(self.sset, self.handles, self.lcps, self.dchar, self.start + start, length)


def _accumulate(stats, st) -> None:
    for f in _lib.STATS_FIELDS:
        setattr(stats, f, getattr(stats, f) + int(getattr(st, f)))


def kway_lcp_merge(streams: list, shared: int = 0, stats=None, cached: bool = False,
                   out_handles: np.ndarray | None = None, out_lcps: np.ndarray | None = None):
    """Merge K sorted runs of one set on the GPU (lcpmerge.py:385-424); more
    than 16 runs merge in rounds of groups of 16 (device.kway_merge_any)."""
    stats = stats if stats is not None else SortStats()
    streams = list(streams)
    n = sum(int(s.length) for s in streams)
    out_h = out_handles if out_handles is not None else np.empty(n, dtype=np.int64)
    out_l = out_lcps if out_lcps is not None else np.empty(n, dtype=np.int64)
    if n == 0:
        return out_h, out_l
    sset = streams[0].sset
    hs = [np.asarray(s.handles[s.start:s.start + s.length], dtype=np.int64) for s in streams]
    ls = [np.asarray(s.lcps[s.start:s.start + s.length], dtype=np.int64) for s in streams]
    off = np.zeros(len(streams) + 1, dtype=np.int64)
    np.cumsum([len(h) for h in hs], out=off[1:])
    h_all = np.concatenate(hs)
    l_all = np.concatenate(ls)
    l_all[off[:-1][off[:-1] < n]] = 0  # a run's first LCP is never read
    ds = D.upload(sset.buffer, h_all)
    l_d = torch.from_numpy(l_all).to(ds.handles.device)
    dchar_d = None
    if cached:
        if all(s.dchar is not None for s in streams):
            dchar_d = torch.from_numpy(np.concatenate(
                [np.asarray(s.dchar[s.start:s.start + s.length], dtype=np.uint8)
                 for s in streams])).to(ds.handles.device)
        else:  # fill_dchar (basecase.py:36-42) on the device
            dchar_d = D.fill_dchar(ds, ds.handles, l_d)
    st = _lib.Stats()
    mh, ml = D.kway_merge_any(ds, off, ds.handles, l_d, dchar_d, shared, st)
    _accumulate(stats, st)
    out_h[:n] = mh.cpu().numpy()
    out_l[:n] = ml.cpu().numpy()
    if out_lcps is None:
        out_l[0] = LCP_UNDEF
    return out_h, out_l


def binary_lcp_merge(a: LcpStream, b: LcpStream, shared: int = 0, stats=None,
                     out_handles: np.ndarray | None = None, out_lcps: np.ndarray | None = None):
    """Merge two sorted runs (lcpmerge.py:143-181) -- the K = 2 merge."""
    return kway_lcp_merge([a, b], shared, stats, False, out_handles, out_lcps)


__all__ = ["LcpStream", "binary_lcp_merge", "kway_lcp_merge"]
