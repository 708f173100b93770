"""Drop-in GPU ``s5_sort`` with the reference signature and return convention.

Mirrors strsort.ssss (ssss.py:361-387): same keyword surface, same
ValueError messages, same return types (``StringSet`` from ``with_handles``,
or ``SortedWithLcp`` with ``lcps[0] = -1``), same ``step_hook(StepRecord)``
protocol (ssss.py:215-224, 340-341).  ``variant``, ``v``, ``seed`` and
``t_medium`` shape only the internal splitter trees and size classes; the
output is the unique stable content order of the input handles, identical
to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as D
from .strset import (
    LCP_UNDEF,
    WORD_CHARS,
    SortedWithLcp,
    SortStats,
    shared_chars,
    word_terminator_pos,
)

DEFAULT_V = 8191
OVERSAMPLE = 2
T_INSERTION = 64
T_MEDIUM = 1 << 20


@dataclass
class SplitterTree:
    """Mirror of strsort.ssss.SplitterTree (ssss.py:37-64)."""

    v: int
    tree: np.ndarray
    inorder: np.ndarray
    node_to_inorder: np.ndarray
    slcp: np.ndarray
    eq_final: np.ndarray
    eq_leftmost: np.ndarray
    term_pos: np.ndarray

    @property
    def depth_levels(self) -> int:
        return int(self.v + 1).bit_length() - 1

    @property
    def num_buckets(self) -> int:
        return 2 * self.v + 1

    @classmethod
    def from_inorder(cls, v: int, inorder: np.ndarray) -> "SplitterTree":
        """Level-order layout and in-order metadata of v sorted splitters."""
        inorder = np.asarray(inorder, dtype=np.uint64)
        L = int(v + 1).bit_length() - 1
        node = np.arange(1, v + 1, dtype=np.int64)
        lvl = np.floor(np.log2(node)).astype(np.int64)
        pos = node - (1 << lvl)
        slot = pos * (1 << (L - lvl)) + (1 << (L - lvl - 1)) - 1
        tree = np.zeros(v + 1, dtype=np.uint64)
        tree[1:] = inorder[slot]
        n2i = np.zeros(v + 1, dtype=np.int64)
        n2i[1:] = slot
        slcp = np.zeros(v + 1, dtype=np.int64)
        if v > 1:
            slcp[1:v] = shared_chars(inorder[:-1], inorder[1:])
        tp = word_terminator_pos(inorder)
        starts = np.r_[True, inorder[1:] != inorder[:-1]]
        eq_leftmost = np.maximum.accumulate(np.where(starts, np.arange(v), 0)).astype(np.int64)
        return cls(v, tree, inorder, n2i, slcp, tp < WORD_CHARS, eq_leftmost, tp)


@dataclass
class StepRecord:
    """Mirror of strsort.ssss.StepRecord (ssss.py:215-224)."""

    lo: int
    hi: int
    depth: int
    bounds: np.ndarray
    child_depths: np.ndarray
    tree: SplitterTree


def child_depths(tree: SplitterTree, depth: int) -> np.ndarray:
    """Eq. 1 prefix credit per bucket (ssss.py:300-307)."""
    k = tree.num_buckets
    depths = np.empty(k, dtype=np.int64)
    depths[0::2] = depth + tree.slcp
    depths[1::2] = depth + tree.term_pos
    return depths


def tree_capacity(n: int, v: int = DEFAULT_V) -> int:
    """Largest 2^d - 1 <= min(v, max(1, n // 2)) (ssss.py:67-73)."""
    limit = min(v, max(1, n // 2))
    d = limit.bit_length()
    while (1 << d) - 1 > limit:
        d -= 1
    return max(1, (1 << d) - 1)


def check_set(buffer, handles: np.ndarray, device_checks_bounds: bool = False) -> None:
    """The reference's input errors (strset.py:70-78).  With
    device_checks_bounds, a buffer that ends in its terminator skips the host
    min/max pass over the handles: s5g_sort_host checks them on the device
    (same ValueError)."""
    n = len(handles)
    if n == 0:
        return
    blen = len(buffer)
    if blen and int(buffer[-1]) == 0 and device_checks_bounds:
        return
    if blen and int(buffer[-1]) == 0:  # the common case: O(1)
        last_zero = blen - 1
    elif isinstance(buffer, np.ndarray):
        z = np.flatnonzero(buffer == 0)
        last_zero = int(z[-1]) if len(z) else -1
    else:
        last_zero = bytes(buffer).rfind(b"\0")
    if last_zero < 0:
        raise ValueError("buffer is not zero-terminated")
    lo, hi = int(handles.min()), int(handles.max())
    if lo < 0 or hi >= blen:
        raise ValueError("handle outside the buffer")
    if hi > last_zero:
        raise ValueError("buffer is not zero-terminated")


class _HookAdapter:
    """ctypes step callback -> step_hook(StepRecord); re-raises hook errors."""

    def __init__(self, hook):
        self.hook = hook
        self.error = None
        self.cb = _lib.STEP_CB(self._call)

    def _call(self, _ctx, lo, hi, depth, v, bounds_p, inorder_p):
        if self.error is not None:
            return
        try:
            bounds = np.ctypeslib.as_array(bounds_p, shape=(2 * v + 2,)).copy()
            inorder = np.ctypeslib.as_array(inorder_p, shape=(v,)).copy()
            tree = SplitterTree.from_inorder(v, inorder)
            self.hook(StepRecord(int(lo), int(hi), int(depth), bounds,
                                 child_depths(tree, int(depth)), tree))
        except BaseException as e:  # surfaced after the library call returns
            self.error = e


def _accumulate(stats, st: _lib.Stats) -> None:
    for f in _lib.STATS_FIELDS:
        setattr(stats, f, getattr(stats, f) + int(getattr(st, f)))


def s5_sort(
    sset,
    depth: int = 0,
    want_lcps: bool = False,
    want_dchar: bool = False,
    variant: str = "unroll",
    v: int = DEFAULT_V,
    seed: int = 1,
    stats=None,
    step_hook=None,
    t_medium: int = T_MEDIUM,
):
    """Sample sort a set on the GPU; with want_lcps returns SortedWithLcp."""
    if variant not in _lib.VARIANTS:
        raise ValueError(f"unknown classify variant: {variant}")
    stats = stats if stats is not None else SortStats()
    handles = np.ascontiguousarray(sset.handles, dtype=np.int64)
    n = len(handles)
    check_set(sset.buffer, handles, device_checks_bounds=step_hook is None)
    if n == 0:
        stats.scratch_words += 0
        out = sset.with_handles(handles.copy())
        if not want_lcps:
            return out
        return SortedWithLcp(out, np.zeros(0, dtype=np.int64),
                             np.zeros(0, dtype=np.uint8) if want_dchar else None, stats)
    st = _lib.Stats()
    if step_hook is None:
        # the end-to-end C-ABI call on the host buffers (s5g_sort_host): the
        # library copies the (pageable or pinned) buffer in, sorts, copies out
        arr = sset.buffer if isinstance(sset.buffer, np.ndarray) else \
            np.frombuffer(sset.buffer, dtype=np.uint8)
        D._require_cuda()
        out_h, lcp_h, dchar_h = D.sort_host(arr, handles, depth=depth, want_lcps=want_lcps,
                                            want_dchar=want_dchar and want_lcps,
                                            variant=variant, v=v, seed=seed,
                                            t_medium=t_medium, stats=st)
        _accumulate(stats, st)
        out = sset.with_handles(out_h)
        if not want_lcps:
            return out
        return SortedWithLcp(out, lcp_h, dchar_h, stats)
    ds = D.upload(sset.buffer, handles)
    hook = _HookAdapter(step_hook)
    out_h, lcps, dchar = D.sort(ds, depth=depth, want_lcps=want_lcps,
                                want_dchar=want_dchar and want_lcps, variant=variant, v=v,
                                seed=seed, t_medium=t_medium, stats=st, step_cb=hook.cb)
    if hook.error is not None:
        raise hook.error
    _accumulate(stats, st)
    out = sset.with_handles(out_h.cpu().numpy())
    if not want_lcps:
        return out
    lcp_h = lcps.cpu().numpy()
    dchar_h = dchar.cpu().numpy() if dchar is not None else None
    return SortedWithLcp(out, lcp_h, dchar_h, stats)


__all__ = [
    "DEFAULT_V", "LCP_UNDEF", "OVERSAMPLE", "SplitterTree", "StepRecord", "T_INSERTION",
    "T_MEDIUM", "child_depths", "s5_sort", "tree_capacity",
]
