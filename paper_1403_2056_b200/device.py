"""Device-side entry: strings resident in HBM, sorted through libs5gpu.so.

PyTorch provides the device buffers and the stream; every byte of sorting
work happens in the library's sm_100a kernels (csrc/s5g.cu).
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import S5G_ARENA_PAD, SortArgs, Stats, check, lib


def _require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1403_2056_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class DeviceStrings:
    """A string set resident on the device: padded arena + int64 handles."""

    arena: torch.Tensor      # uint8, arena_len + pad bytes, pad zeroed
    arena_len: int
    handles: torch.Tensor    # int64[n]
    # terminators before each 64-byte block (s5g_load_delimited_rank), when
    # the handles are the arena's string starts: start -> index without a search
    rank64: torch.Tensor | None = None

    @property
    def n(self) -> int:
        return int(self.handles.numel())


def alloc_arena(arena_len: int, device) -> torch.Tensor:
    cap = (arena_len + S5G_ARENA_PAD + 15) // 16 * 16
    a = torch.empty(cap, dtype=torch.uint8, device=device)
    a[arena_len:].zero_()
    return a


def upload(buffer, handles, device=None) -> DeviceStrings:
    """Copy a host buffer (bytes / uint8 array) and handles into HBM."""
    device = device or _require_cuda()
    arr = buffer if isinstance(buffer, np.ndarray) else np.frombuffer(buffer, dtype=np.uint8)
    alen = int(arr.size)
    arena = alloc_arena(alen, device)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # read-only bytes buffers are only read
        if alen:
            arena[:alen].copy_(torch.from_numpy(arr), non_blocking=False)
        h = torch.from_numpy(np.ascontiguousarray(handles, dtype=np.int64))
    return DeviceStrings(arena, alen, h.to(device))


def workspace_bytes(n: int, t_medium: int) -> int:
    return int(lib().s5g_workspace_bytes(n, t_medium))


def sort(ds: DeviceStrings, depth: int = 0, want_lcps: bool = True, want_dchar: bool = False,
         variant: str = "unroll", v: int = 8191, seed: int = 1, t_medium: int = 1 << 20,
         stats: Stats | None = None, step_cb=None, out=None, workspace=None):
    """Sort device strings; returns (out_handles, lcps | None, dchar | None) tensors."""
    if variant not in _lib.VARIANTS:
        raise ValueError(f"unknown classify variant: {variant}")
    n = ds.n
    dev = ds.handles.device
    out_h = out[0] if out is not None else torch.empty(n, dtype=torch.int64, device=dev)
    lcps = None
    if want_lcps or want_dchar:
        lcps = out[1] if out is not None else torch.empty(n, dtype=torch.int64, device=dev)
    dchar = torch.empty(n, dtype=torch.uint8, device=dev) if want_dchar else None
    wsb = workspace_bytes(n, t_medium)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    a = SortArgs()
    a.arena = ds.arena.data_ptr()
    a.arena_len = ds.arena_len
    a.handles = ds.handles.data_ptr()
    a.n = n
    a.depth = depth
    a.out_handles = out_h.data_ptr()
    a.out_lcps = lcps.data_ptr() if lcps is not None else None
    a.out_dchar = dchar.data_ptr() if dchar is not None else None
    a.workspace = workspace.data_ptr()
    a.workspace_bytes = workspace.numel()
    a.stream = torch.cuda.current_stream(dev).cuda_stream
    a.variant = _lib.VARIANTS[variant]
    a.v = int(max(1, min(v, 8191)))
    a.seed = int(seed) & ((1 << 64) - 1)
    a.t_medium = int(t_medium)
    st = stats if stats is not None else Stats()
    a.stats = C.pointer(st)
    a.step_cb = step_cb if step_cb is not None else _lib.STEP_CB()
    a.step_ctx = None
    check(lib().s5g_sort(C.byref(a)))
    return out_h, lcps, dchar


def extract_keys(ds: DeviceStrings, depth: int) -> torch.Tensor:
    out = torch.empty(ds.n, dtype=torch.int64, device=ds.handles.device)
    check(lib().s5g_extract_keys(ds.arena.data_ptr(), ds.arena_len, ds.handles.data_ptr(),
                                 ds.n, depth, out.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream))
    return out


def select_splitters(sample: torch.Tensor, v: int):
    """Device select_splitters: (tree[v+1], inorder[v], term_pos[v], eq_bucket[v+1])."""
    dev = sample.device
    tree = torch.empty(v + 1, dtype=torch.int64, device=dev)
    inorder = torch.empty(v, dtype=torch.int64, device=dev)
    tpos = torch.empty(v, dtype=torch.uint8, device=dev)
    eqb = torch.empty(v + 1, dtype=torch.int16, device=dev)
    check(lib().s5g_select_splitters(sample.data_ptr(), sample.numel(), v, tree.data_ptr(),
                                     inorder.data_ptr(), tpos.data_ptr(), eqb.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
    return tree, inorder, tpos, eqb


def classify(keys: torch.Tensor, tree: torch.Tensor, eq_bucket: torch.Tensor, v: int,
             variant: str = "unroll") -> torch.Tensor:
    if variant not in _lib.VARIANTS:
        raise ValueError(f"unknown classify variant: {variant}")
    out = torch.empty(keys.numel(), dtype=torch.int16, device=keys.device)
    check(lib().s5g_classify(keys.data_ptr(), keys.numel(), tree.data_ptr(),
                             eq_bucket.data_ptr(), v, _lib.VARIANTS[variant], out.data_ptr(),
                             torch.cuda.current_stream().cuda_stream))
    return out


def fill_dchar(ds: DeviceStrings, sorted_handles: torch.Tensor, lcps: torch.Tensor) -> torch.Tensor:
    out = torch.empty(sorted_handles.numel(), dtype=torch.uint8, device=sorted_handles.device)
    check(lib().s5g_fill_dchar(ds.arena.data_ptr(), sorted_handles.data_ptr(), lcps.data_ptr(),
                               sorted_handles.numel(), out.data_ptr(),
                               torch.cuda.current_stream().cuda_stream))
    return out


def sort_host(buffer, handles, depth: int = 0, want_lcps: bool = True, want_dchar: bool = False,
              variant: str = "unroll", v: int = 8191, seed: int = 1, t_medium: int = 1 << 20,
              stats: Stats | None = None, out_handles=None, out_lcps=None):
    """End-to-end C-ABI call on host buffers (s5g_sort_host)."""
    if variant not in _lib.VARIANTS:
        raise ValueError(f"unknown classify variant: {variant}")
    arr = buffer if isinstance(buffer, np.ndarray) else np.frombuffer(buffer, dtype=np.uint8)
    h = handles if isinstance(handles, np.ndarray) else np.asarray(handles, dtype=np.int64)
    n = len(h)
    oh = out_handles if out_handles is not None else np.empty(n, dtype=np.int64)
    ol = out_lcps if out_lcps is not None else (np.empty(n, dtype=np.int64) if want_lcps else None)
    od = np.empty(n, dtype=np.uint8) if want_dchar else None
    st = stats if stats is not None else Stats()
    ptr = lambda x: x.ctypes.data if x is not None and x.size else None  # noqa: E731
    check(lib().s5g_sort_host(ptr(arr), arr.size, ptr(h), n, depth, ptr(oh), ptr(ol), ptr(od),
                              _lib.VARIANTS[variant], int(min(max(v, 1), 8191)), int(seed),
                              int(t_medium), C.byref(st)))
    return oh, ol, od


def partition(ds: DeviceStrings, base_index: int, splitters: list[bytes], splitter_gidx,
              string_gidx: torch.Tensor | None = None) -> torch.Tensor:
    """Destination rank of every string (s5g_partition); splitters sorted.
    A string's global index is string_gidx[i], else base_index + i."""
    dev = ds.handles.device
    blob = b"".join(splitters)
    off = np.zeros(len(splitters) + 1, dtype=np.int64)
    if splitters:
        np.cumsum([len(x) for x in splitters], out=off[1:])
    blob_d = torch.from_numpy(np.frombuffer(blob, dtype=np.uint8).copy() if blob else
                              np.zeros(1, np.uint8)).to(dev)
    off_d = torch.from_numpy(off).to(dev)
    gidx_d = torch.as_tensor(np.asarray(splitter_gidx, dtype=np.int64), device=dev)
    out = torch.empty(ds.n, dtype=torch.int32, device=dev)
    check(lib().s5g_partition(ds.arena.data_ptr(), ds.arena_len, ds.handles.data_ptr(), ds.n,
                              int(base_index),
                              string_gidx.data_ptr() if string_gidx is not None else None,
                              blob_d.data_ptr(), off_d.data_ptr(),
                              gidx_d.data_ptr() if len(splitters) else None, len(splitters),
                              out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    return out


def lengths(ds: DeviceStrings) -> torch.Tensor:
    out = torch.empty(ds.n, dtype=torch.int64, device=ds.handles.device)
    check(lib().s5g_lengths(ds.arena.data_ptr(), ds.arena_len, ds.handles.data_ptr(), ds.n,
                            out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return out


def pack(ds: DeviceStrings, handles: torch.Tensor, lens: torch.Tensor, dst_off: torch.Tensor,
         total: int) -> torch.Tensor:
    dst = torch.empty(max(total, 1), dtype=torch.uint8, device=ds.handles.device)
    check(lib().s5g_pack(ds.arena.data_ptr(), ds.arena_len, handles.data_ptr(), lens.data_ptr(),
                         dst_off.data_ptr(), handles.numel(), dst.data_ptr(),
                         torch.cuda.current_stream().cuda_stream))
    return dst


def load_delimited(data, delimiter: int = 0, device=None) -> DeviceStrings:
    """load_delimited (strset.py:113-134) with the scan on the GPU: the bytes
    are copied to HBM once and become the arena in place."""
    if not (0 <= delimiter < 256):
        raise ValueError("delimiter must be a byte value")
    device = device or _require_cuda()
    arr = data if isinstance(data, np.ndarray) else np.frombuffer(data, dtype=np.uint8)
    L = int(arr.size)
    if L == 0:
        return DeviceStrings(alloc_arena(0, device), 0, torch.zeros(0, dtype=torch.int64, device=device))
    # the reference appends a terminator unless the input already ends in the
    # delimiter (after remapping); the arena gets room for one more byte
    ends = int(arr[-1]) == delimiter
    alen = L if ends else L + 1
    arena = alloc_arena(alen, device)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        arena[:L].copy_(torch.from_numpy(arr))
    if not ends:
        arena[L] = delimiter  # the appended terminator (remapped to 0 with the rest)
    handles = torch.empty(alen + 1, dtype=torch.int64, device=device)
    nchunks = (alen + 16384 - 1) // 16384
    ws = torch.empty(16 + 4 * nchunks, dtype=torch.uint8, device=device)
    n = C.c_int64()
    check(lib().s5g_load_delimited(arena.data_ptr(), alen, delimiter, handles.data_ptr(),
                                   C.byref(n), ws.data_ptr(), ws.numel(),
                                   torch.cuda.current_stream(device).cuda_stream))
    return DeviceStrings(arena, alen, handles[: n.value])


def dist_stats(lcps: torch.Tensor) -> tuple[int, int]:
    """(D, L) of a sorted set from its exact LCP array (strset.py:290-309)."""
    D, L = C.c_int64(), C.c_int64()
    check(lib().s5g_dist_stats(lcps.data_ptr(), lcps.numel(), C.byref(D), C.byref(L),
                               torch.cuda.current_stream(lcps.device).cuda_stream))
    return int(D.value), int(L.value)


def kway_merge(ds: DeviceStrings, run_offsets, handles: torch.Tensor, lcps: torch.Tensor,
               dchar: torch.Tensor | None = None, shared: int = 0, stats: Stats | None = None):
    """Stable K-way LCP merge of sorted runs laid end to end in handles/lcps
    (run j = [run_offsets[j], run_offsets[j+1])); s5g_kway_merge.  Returns
    (out_handles, out_lcps) with out_lcps[0] = shared."""
    off = np.ascontiguousarray(run_offsets, dtype=np.int64)
    k = len(off) - 1
    n = int(off[-1] - off[0])
    dev = handles.device
    out_h = torch.empty(n, dtype=torch.int64, device=dev)
    out_l = torch.empty(n, dtype=torch.int64, device=dev)
    wsb = int(lib().s5g_merge_workspace_bytes(n, max(k, 1)))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    st = stats if stats is not None else Stats()
    check(lib().s5g_kway_merge(ds.arena.data_ptr(), ds.arena_len, k,
                               off.ctypes.data_as(C.POINTER(C.c_int64)), handles.data_ptr(),
                               lcps.data_ptr(), dchar.data_ptr() if dchar is not None else None,
                               int(shared), out_h.data_ptr(), out_l.data_ptr(), ws.data_ptr(),
                               ws.numel(), torch.cuda.current_stream(dev).cuda_stream,
                               C.byref(st)))
    return out_h, out_l


def kway_merge_any(ds: DeviceStrings, run_offsets, handles: torch.Tensor, lcps: torch.Tensor,
                   dchar: torch.Tensor | None = None, shared: int = 0,
                   stats: Stats | None = None):
    """kway_merge for any number of runs: while there are more than 16, merge
    consecutive groups of up to 16 (ties to the earlier run, so the result
    stays the stable order) and repeat -- the reference's kway_lcp_merge /
    partitioned_merge_sort take any K (lcpmerge.py:385-424,
    parallel.py:885-994)."""
    off = np.ascontiguousarray(run_offsets, dtype=np.int64)
    while len(off) - 1 > 16:
        K = len(off) - 1
        out_h = torch.empty_like(handles)
        out_l = torch.empty_like(lcps)
        new_off = [int(off[0])]
        for g0 in range(0, K, 16):
            g1 = min(K, g0 + 16)
            lo, hi = int(off[g0] - off[0]), int(off[g1] - off[0])
            if g1 - g0 == 1 or hi == lo:
                out_h[lo:hi] = handles[lo:hi]
                out_l[lo:hi] = lcps[lo:hi]
            else:
                mh, ml = kway_merge(ds, off[g0:g1 + 1] - off[g0], handles[lo:hi], lcps[lo:hi],
                                    dchar[lo:hi] if dchar is not None else None, shared, stats)
                out_h[lo:hi] = mh
                out_l[lo:hi] = ml
            new_off.append(int(off[g1]))
        handles, lcps = out_h, out_l
        if dchar is not None:  # distinguishing characters of the merged runs
            dchar = fill_dchar(ds, handles, lcps.clamp(min=0))
        off = np.asarray(new_off, dtype=np.int64)
    return kway_merge(ds, off, handles, lcps, dchar, shared, stats)


def group_by_dest(dest: torch.Tensor, G: int):
    """Stable order of the strings by destination rank and the per-rank
    counts (s5g_group_by_dest)."""
    n = dest.numel()
    dev = dest.device
    d = dest.to(torch.int32).contiguous()
    order = torch.empty(n, dtype=torch.int64, device=dev)
    counts = torch.empty(G, dtype=torch.int64, device=dev)
    ws = torch.empty(max(int(lib().s5g_group_workspace_bytes(n, G)), 1), dtype=torch.uint8, device=dev)
    check(lib().s5g_group_by_dest(d.data_ptr(), n, G, order.data_ptr(), counts.data_ptr(),
                                  ws.data_ptr(), ws.numel(), torch.cuda.current_stream(dev).cuda_stream))
    return order, counts


def positions(handles: torch.Tensor, query: torch.Tensor, map_len: int) -> torch.Tensor:
    """Input position of every query handle (unique handles < map_len): s5g_positions."""
    dev = handles.device
    out = torch.empty(query.numel(), dtype=torch.int64, device=dev)
    mp = torch.empty(max(map_len, 1), dtype=torch.int32, device=dev)
    check(lib().s5g_positions(handles.data_ptr(), handles.numel(), query.data_ptr(), query.numel(),
                              mp.data_ptr(), map_len, out.data_ptr(),
                              torch.cuda.current_stream(dev).cuda_stream))
    return out


def input_positions(in_handles: torch.Tensor, out_handles: torch.Tensor, max_handle: int) -> torch.Tensor:
    """Input position of every sorted handle of a stable sort's output
    (s5g_input_positions: two stable radix sorts by handle; repeated handles
    -- the same string -- are matched in input order)."""
    n = in_handles.numel()
    dev = in_handles.device
    out = torch.empty(n, dtype=torch.int64, device=dev)
    if n == 0:
        return out
    ws = torch.empty(int(lib().s5g_input_positions_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    check(lib().s5g_input_positions(in_handles.data_ptr(), out_handles.data_ptr(), n,
                                    int(max(max_handle, 1)), out.data_ptr(), ws.data_ptr(),
                                    ws.numel(), torch.cuda.current_stream(dev).cuda_stream))
    return out


def rank_positions(ds: DeviceStrings, query: torch.Tensor) -> torch.Tensor:
    """Index of the string starting at each query handle, for an arena loaded
    with its rank directory (s5g_rank_positions)."""
    m = query.numel()
    out = torch.empty(m, dtype=torch.int64, device=query.device)
    if m:
        check(lib().s5g_rank_positions(ds.arena.data_ptr(), ds.arena_len, ds.rank64.data_ptr(),
                                       query.contiguous().data_ptr(), m, out.data_ptr(),
                                       torch.cuda.current_stream(query.device).cuda_stream))
    return out


def gather_i64(src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """src[idx] for int64 device arrays (s5g_gather_i64)."""
    out = torch.empty(idx.numel(), dtype=torch.int64, device=src.device)
    if idx.numel():
        check(lib().s5g_gather_i64(src.data_ptr(), idx.contiguous().data_ptr(), idx.numel(),
                                   out.data_ptr(), torch.cuda.current_stream(src.device).cuda_stream))
    return out


def pack_order(ds: DeviceStrings, order: torch.Tensor, counts: list[int]):
    """The exchange's send buffer: strings handles[order[k]] (with their
    terminators) back to back, and the bytes per destination
    (s5g_pack_plan + s5g_pack)."""
    n = order.numel()
    dev = ds.handles.device
    G = len(counts)
    cnt = torch.tensor(counts, dtype=torch.int64, device=dev)
    h = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    dest = torch.empty(G, dtype=torch.int64, device=dev)
    ws = torch.empty(int(lib().s5g_pack_plan_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    check(lib().s5g_pack_plan(ds.arena.data_ptr(), ds.arena_len, ds.handles.data_ptr(),
                              order.contiguous().data_ptr() if n else None, n, cnt.data_ptr(), G,
                              h.data_ptr(), off.data_ptr(), dest.data_ptr(), ws.data_ptr(),
                              ws.numel(), st))
    dest_h = dest.cpu().tolist()
    total = int(sum(dest_h))
    payload = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    if n:
        check(lib().s5g_pack(ds.arena.data_ptr(), ds.arena_len, h.data_ptr(), None, off.data_ptr(),
                             n, payload.data_ptr(), st))
    return payload[:total], [int(x) for x in dest_h]
