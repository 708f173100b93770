"""Multi-GPU S^5: one process per GPU, sample-sort partition + all-to-all.

The reference's fully parallel step (``_ParallelS5Run._phased_step``,
parallel.py:359-398: sample -> splitters -> classify per shard -> interleaved
prefix sum -> scatter) lifted to G ranks:

1. every rank samples strings of its shard; the samples are all-gathered and
   every rank picks the same G-1 *string* splitters (byte prefixes of sampled
   strings, capped at ``max_splitter_len``) with a (string, global index)
   tie-break -- so equal strings split by input position and the result stays
   the stable order;
2. classify: destination rank of every string (``s5g_partition`` on the GPU);
3. exchange counts, then the strings' bytes and global input indices with
   one all-to-all (NCCL over NVLink; ``packed`` mode) -- or only the handles
   when every rank holds the whole arena (``replicated`` mode, e.g. a suffix
   set's text);
4. local S^5 sort of the received strings (they arrive in global input order,
   so the local stable sort is the global stable order);
5. boundary-LCP fix-up: each rank gets the last string of the previous
   non-empty rank and sets ``lcps[0]`` (rank 0 keeps -1) -- the analogue of
   ``_boundary_lcps`` (parallel.py:447-455) and the merge-boundary recompute
   of partitioned_merge_sort (parallel.py:989-991).

The concatenation of the ranks' outputs is the reference's output.

``distributed_merge_sort`` is the other strategy (SURVEY 8f row 1,
partitioned_merge_sort): sort first, then cut the sorted runs at sampled
splitters, exchange the sorted pieces with their LCPs and distinguishing
characters, and K-way LCP merge them on every rank.

Compute is pluggable (``backend``): ``GpuBackend`` runs every step in the
sm_100a library; tests substitute a CPU backend to run the collective logic
on ``gloo`` without a GPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

LCP_UNDEF = -1


@dataclass
class Shard:
    """One rank's input: a zero-terminated buffer, handles into it, and the
    global input index of its first string."""

    buffer: object          # np.ndarray[uint8] (host) -- the backend uploads it
    handles: np.ndarray     # int64
    base_index: int


@dataclass
class DistResult:
    gidx: torch.Tensor      # global input index of every string this rank holds, sorted
    lcps: torch.Tensor | None
    arena: object           # the rank-local arena the strings live in
    handles: torch.Tensor   # sorted handles into `arena`
    n_total: int


def _alltoallv(send: torch.Tensor, send_counts: list[int], recv_counts: list[int], group,
               out: torch.Tensor | None = None):
    """Variable-size all-to-all of a 1-D tensor (NCCL all_to_all_single;
    point-to-point pairs on backends without all-to-all, e.g. gloo).  `out`:
    receive in place (sum(recv_counts) elements), e.g. straight into the
    arena the received strings will live in."""
    G = dist.get_world_size(group)
    r = dist.get_rank(group)
    recv = out if out is not None else torch.empty(sum(recv_counts), dtype=send.dtype,
                                                   device=send.device)
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(recv, send, recv_counts, send_counts, group=group)
        return recv
    so = np.r_[0, np.cumsum(send_counts)]
    ro = np.r_[0, np.cumsum(recv_counts)]
    recv[ro[r]:ro[r + 1]] = send[so[r]:so[r + 1]]
    reqs = []
    for k in range(1, G):
        dst, src = (r + k) % G, (r - k) % G
        if send_counts[dst]:
            reqs.append(dist.isend(send[so[dst]:so[dst + 1]].contiguous(), dst, group=group))
        if recv_counts[src]:
            buf = torch.empty(recv_counts[src], dtype=send.dtype, device=send.device)
            reqs.append((dist.irecv(buf, src, group=group), buf, ro[src]))
    for q in reqs:
        if isinstance(q, tuple):
            q[0].wait()
            recv[q[2]:q[2] + len(q[1])] = q[1]
        else:
            q.wait()
    return recv


def _all_gather_strings(items: list[tuple[bytes, int]], device, group) -> list[tuple[bytes, int]]:
    """All-gather every rank's (string, global index) list through plain
    tensors (NCCL / gloo buffers, no pickling): counts first, then one
    fixed-width record per string -- [length, index, bytes padded to the
    longest string of the job]."""
    G = dist.get_world_size(group)
    k = torch.tensor([len(items), max((len(b) for b, _ in items), default=0)],
                     dtype=torch.int64, device=device)
    ks = [torch.empty_like(k) for _ in range(G)]
    dist.all_gather(ks, k, group=group)
    ks = torch.stack(ks).cpu().tolist()  # one device read for all ranks' counts
    kmax = max(x[0] for x in ks)
    width = max(x[1] for x in ks)
    if kmax == 0:
        return []
    rec = 16 + width
    # records built and taken apart with whole-array operations (a numpy call
    # per string cost ~3 ms per gather of 1024 samples)
    buf = np.zeros((kmax, rec), dtype=np.uint8)
    if items:
        k_mine = len(items)
        meta = np.empty((k_mine, 2), dtype=np.int64)
        meta[:, 0] = [len(b) for b, _ in items]
        meta[:, 1] = [g for _, g in items]
        buf[:k_mine, :16] = meta.view(np.uint8).reshape(k_mine, 16)
        if width:
            body = b"".join(b.ljust(width, b"\0") for b, _ in items)
            buf[:k_mine, 16:] = np.frombuffer(body, dtype=np.uint8).reshape(k_mine, width)
    t = torch.from_numpy(buf.reshape(-1)).to(device)
    out = torch.empty(G * t.numel(), dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(out, t, group=group) if dist.get_backend(group) == "nccl" else \
        dist.all_gather(list(out.view(G, -1).unbind(0)), t, group=group)
    allrec = out.cpu().numpy().reshape(G, kmax, rec)
    res = []
    for q in range(G):
        kq = ks[q][0]
        if not kq:
            continue
        a = allrec[q, :kq]
        meta = np.ascontiguousarray(a[:, :16]).view(np.int64)
        body = np.ascontiguousarray(a[:, 16:]).tobytes()
        lens, gs = meta[:, 0].tolist(), meta[:, 1].tolist()
        res.extend((body[i * width: i * width + lens[i]], gs[i]) for i in range(kq))
    return res


def sample_positions(n: int, k: int, seed: int, rank: int) -> np.ndarray:
    """k uniformly random positions of a shard of n strings (seeded by
    (seed, rank); draw_sample's role, ssss.py:76-82, at the partition level)
    -- regular positions of an unsorted shard would follow its input order."""
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    rng = np.random.default_rng((seed, rank, n))
    return np.unique(rng.integers(0, n, size=min(k, n), dtype=np.int64))


def pick_splitters(samples: list[tuple[bytes, int]], G: int) -> tuple[list[bytes], list[int]]:
    """G-1 equally spaced splitters from the sorted (string, global index) samples."""
    samples = sorted(samples)
    if not samples:
        return [], []
    picks = [samples[(k * len(samples)) // G] for k in range(1, G)]
    return [p[0] for p in picks], [p[1] for p in picks]


def distributed_sort(shard: Shard, backend, group=None, samples_per_rank: int = 1024,
                     max_splitter_len: int = 64, want_lcps: bool = True,
                     mode: str = "packed", seed: int = 1, stats: dict | None = None,
                     **sort_kw) -> DistResult:
    """Globally stable sort of the union of all ranks' shards (see module doc)."""
    G = dist.get_world_size(group)
    r = dist.get_rank(group)
    local = backend.prepare(shard)
    n_local = len(shard.handles)
    # 1. samples -> identical splitters on every rank
    mine = backend.sample(local, shard, samples_per_rank, max_splitter_len, seed=seed, rank=r)
    sp, sp_g = pick_splitters(_all_gather_strings(mine, backend.comm_device, group), G)
    # 2. destination rank of every local string (stable within a destination)
    dest = backend.partition(local, shard, sp, sp_g)
    order, counts = backend.group_by_dest(dest, G)
    # 3. exchange
    cnt = torch.tensor(counts, dtype=torch.int64, device=backend.comm_device)
    rcnt = torch.empty_like(cnt)
    dist.all_to_all_single(rcnt, cnt, group=group) if dist.get_backend(group) == "nccl" else \
        _gather_counts(cnt, rcnt, group)
    recv_counts = [int(x) for x in rcnt.tolist()]
    gidx_send = backend.global_index(shard, order)
    gidx = _alltoallv(gidx_send, counts, recv_counts, group)
    if mode == "replicated":
        h_send = backend.take_handles(local, order)
        handles = _alltoallv(h_send, counts, recv_counts, group)
        arena = local
    elif mode == "packed":
        payload, byte_counts = backend.pack(local, order, counts)
        bcnt = torch.tensor(byte_counts, dtype=torch.int64, device=backend.comm_device)
        rbcnt = torch.empty_like(bcnt)
        dist.all_to_all_single(rbcnt, bcnt, group=group) if dist.get_backend(group) == "nccl" else \
            _gather_counts(bcnt, rbcnt, group)
        rb = [int(x) for x in rbcnt.tolist()]
        # received straight into the arena the strings will live in, when the
        # backend offers one (no second copy of the shard)
        into = backend.recv_arena(sum(rb)) if hasattr(backend, "recv_arena") else None
        rbytes = _alltoallv(payload, byte_counts, rb, group, out=into)
        del payload
        arena, handles = backend.unpack(rbytes, sum(recv_counts)) if into is not None else \
            backend.unpack(rbytes)
        if stats is not None:  # bytes this rank sends to other ranks (NVLink traffic)
            stats["sent_bytes"] = int(sum(b for q, b in enumerate(byte_counts) if q != r) +
                                      24 * sum(c for q, c in enumerate(counts) if q != r))
    else:
        raise ValueError(f"unknown exchange mode: {mode}")
    # 4. local sort: received in global input order -> stable local sort
    perm, lcps = backend.local_sort(arena, handles, want_lcps, **sort_kw)
    sorted_h = backend.sorted_handles(handles, perm) if hasattr(backend, "sorted_handles") else \
        backend.take(handles, perm)
    sorted_g = backend.take(gidx, perm)
    # 5. LCP at the rank boundary
    if want_lcps:
        _boundary_lcp(backend, arena, sorted_h, lcps, G, r, group)
    total = torch.tensor([n_local], dtype=torch.int64, device=backend.comm_device)
    dist.all_reduce(total, group=group)
    return DistResult(sorted_g, lcps, arena, sorted_h, int(total.item()))


def _exchange_counts(counts: list[int], device, group) -> list[int]:
    cnt = torch.tensor(counts, dtype=torch.int64, device=device)
    rcnt = torch.empty_like(cnt)
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(rcnt, cnt, group=group)
    else:
        _gather_counts(cnt, rcnt, group)
    return [int(x) for x in rcnt.tolist()]


def _boundary_lcp(backend, arena, sorted_h, lcps, G, r, group):
    """lcps[0] of this rank against the last string of the previous
    non-empty rank (rank 0 keeps -1): _boundary_lcps, parallel.py:447-455."""
    first = backend.string_bytes(arena, sorted_h[:1]) if len(sorted_h) else None
    last = backend.string_bytes(arena, sorted_h[-1:]) if len(sorted_h) else None
    # every rank's last string (rank q -> global index q marks it), no pickling
    got = dict((g, b) for b, g in _all_gather_strings([] if last is None else [(last, r)],
                                                      backend.comm_device, group))
    ends = [got.get(q) for q in range(G)]
    prev = next((ends[q] for q in range(r - 1, -1, -1) if ends[q] is not None), None)
    if len(sorted_h):
        lcps[0] = LCP_UNDEF if prev is None else _lcp_bytes(prev, first)


def distributed_merge_sort(shard: Shard, backend, group=None, samples_per_rank: int = 1024,
                           max_splitter_len: int = 64, use_cache: bool = True,
                           **sort_kw) -> DistResult:
    """partitioned_merge_sort (parallel.py:885-994) across G ranks: every rank
    sorts its shard (S^5 with LCPs and distinguishing characters), the sorted
    runs are cut at G-1 regularly sampled string splitters (ties by global
    index), each rank receives one sorted piece from every rank -- strings,
    global indices, LCPs, characters -- and K-way LCP merges them
    (s5g_kway_merge, cached comparisons when use_cache; pieces arrive in rank
    order = input order, so merge ties keep the stable order).  Same result
    as distributed_sort; the exchange moves the sorted runs instead of the
    raw shard."""
    G = dist.get_world_size(group)
    r = dist.get_rank(group)
    local = backend.prepare(shard)
    n_local = len(shard.handles)
    hnd = backend.handles_of(local, shard)
    perm, lcps = backend.local_sort(local, hnd, True, **sort_kw)
    sorted_h = backend.take(hnd, perm)
    gidx = perm.to(torch.int64) + shard.base_index
    # 1. regular samples of the sorted run -> identical splitters everywhere
    mine = backend.sample_run(local, sorted_h, gidx, samples_per_rank, max_splitter_len)
    sp, sp_g = pick_splitters(_all_gather_strings(mine, backend.comm_device, group), G)
    # 2. cut the sorted run (destinations are non-decreasing along it)
    dest = backend.partition(local, shard, sp, sp_g, handles=sorted_h, gidx=gidx)
    counts = backend.dest_counts(dest, G) if n_local else [0] * G
    recv_counts = _exchange_counts(counts, backend.comm_device, group)
    # 3. exchange the sorted pieces
    gidx_r = _alltoallv(gidx.to(backend.comm_device), counts, recv_counts, group)
    lcp_r = _alltoallv(lcps.to(backend.comm_device), counts, recv_counts, group)
    dchar_r = None
    if use_cache:
        dchar = backend.fill_dchar(local, sorted_h, lcps)
        dchar_r = _alltoallv(dchar.to(backend.comm_device), counts, recv_counts, group)
    payload, byte_counts = backend.pack(local, perm, counts)
    rbyte_counts = _exchange_counts(byte_counts, backend.comm_device, group)
    rbytes = _alltoallv(payload, byte_counts, rbyte_counts, group)
    arena, starts = backend.unpack(rbytes)
    # 4. K-way LCP merge of the G received runs
    run_off = np.r_[0, np.cumsum(recv_counts)].astype(np.int64)
    mh, ml = backend.kway_merge(arena, run_off, starts, lcp_r, dchar_r)
    pos = backend.positions(arena, starts, mh)
    out_g = backend.take(gidx_r, pos)
    # 5. LCP at the rank boundary
    _boundary_lcp(backend, arena, mh, ml, G, r, group)
    total = torch.tensor([n_local], dtype=torch.int64, device=backend.comm_device)
    dist.all_reduce(total, group=group)
    return DistResult(out_g, ml, arena, mh, int(total.item()))


def handle_positions(handles: torch.Tensor, out_h: torch.Tensor) -> torch.Tensor:
    """Input position of every sorted handle (handles unique; in packed mode
    they are increasing string starts)."""
    srt, inv = torch.sort(handles)
    return inv[torch.searchsorted(srt, out_h)]


def _gather_counts(cnt: torch.Tensor, out: torch.Tensor, group) -> None:
    G = dist.get_world_size(group)
    r = dist.get_rank(group)
    rows = [torch.empty_like(cnt) for _ in range(G)]
    dist.all_gather(rows, cnt, group=group)
    for q in range(G):
        out[q] = rows[q][r]


def _lcp_bytes(a: bytes, b: bytes) -> int:
    i = 0
    while i < len(a) and i < len(b) and a[i] == b[i]:
        i += 1
    return i


class GpuBackend:
    """Every compute step in libs5gpu.so (sm_100a); collectives over NCCL."""

    def __init__(self, device=None):
        self.comm_device = device or torch.device("cuda", torch.cuda.current_device())

    def prepare(self, shard: Shard):
        from . import device as D

        if isinstance(shard.buffer, D.DeviceStrings):  # already resident in HBM
            return shard.buffer
        return D.upload(shard.buffer, shard.handles, self.comm_device)

    def sample(self, ds, shard: Shard, k: int, maxlen: int, seed: int = 1, rank: int = 0):
        """k random strings of the shard (prefixes <= maxlen) with their
        global indices; the strings are packed on the device."""
        from . import device as D

        pos = sample_positions(ds.n, k, seed, rank)
        if len(pos) == 0:
            return []
        order = torch.as_tensor(pos, device=ds.handles.device)
        return self._strings(ds, order, [int(shard.base_index + p) for p in pos], maxlen)

    def _strings(self, ds, order, gidx, maxlen):
        from . import device as D

        payload, _ = D.pack_order(ds, order, [int(order.numel())])
        raw = payload.cpu().numpy().tobytes()
        out = raw.split(b"\0")[: len(gidx)]
        return [(x[:maxlen], g) for x, g in zip(out, gidx)]

    def take(self, src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
        from . import device as D

        return D.gather_i64(src, idx)

    def partition(self, ds, shard: Shard, sp, sp_g, handles=None, gidx=None):
        from . import device as D

        if handles is not None:
            ds = D.DeviceStrings(ds.arena, ds.arena_len, handles)
        return D.partition(ds, shard.base_index, sp, sp_g, gidx)

    def handles_of(self, ds, shard: Shard):
        return ds.handles

    def dest_counts(self, dest: torch.Tensor, G: int) -> list[int]:
        return self.group_by_dest(dest, G)[1]

    def positions(self, ds, handles: torch.Tensor, query: torch.Tensor) -> torch.Tensor:
        from . import device as D

        return D.input_positions(handles, query, ds.arena_len)

    def sample_run(self, ds, handles, gidx, k: int, maxlen: int):
        """Equally spaced strings of a sorted run (prefixes <= maxlen) with
        their global indices (regular sampling of a sorted run, the merge
        strategy's splitters)."""
        from . import device as D

        n = handles.numel()
        if n == 0:
            return []
        pos = torch.as_tensor(np.unique(np.linspace(0, n - 1, num=min(k, n)).astype(np.int64)),
                              device=handles.device)
        sub = D.DeviceStrings(ds.arena, ds.arena_len, handles)
        return self._strings(sub, pos, [int(x) for x in D.gather_i64(gidx, pos).cpu().tolist()],
                             maxlen)

    def fill_dchar(self, ds, sorted_h, lcps):
        from . import device as D

        return D.fill_dchar(ds, sorted_h, lcps)

    def kway_merge(self, ds, run_off, handles, lcps, dchar):
        from . import device as D

        return D.kway_merge(ds, run_off, handles, lcps, dchar, 0)

    def group_by_dest(self, dest: torch.Tensor, G: int):
        from . import device as D

        order, counts = D.group_by_dest(dest, G)  # stable counting sort (s5g_group_by_dest)
        return order, counts.tolist()

    def global_index(self, shard: Shard, order: torch.Tensor):
        return order.to(torch.int64) + shard.base_index

    def take_handles(self, ds, order):
        from . import device as D

        return D.gather_i64(ds.handles, order)

    def pack(self, ds, order, counts):
        """Send buffer in destination order and bytes per destination, all
        in library kernels (s5g_pack_plan + s5g_pack)."""
        from . import device as D

        return D.pack_order(ds, order, list(counts))

    def recv_arena(self, nbytes: int) -> torch.Tensor:
        """A padded arena for nbytes of received strings; the all-to-all
        writes into the returned view and `unpack` adopts it without a copy."""
        from . import device as D

        self._recv = D.alloc_arena(nbytes, self.comm_device)
        return self._recv[:nbytes]

    def unpack(self, rbytes: torch.Tensor, n_strings: int | None = None):
        """Received zero-terminated strings -> arena + string starts
        (s5g_load_delimited_n with delimiter 0).  n_strings: how many strings
        arrived (known from the index exchange), so the starts need
        n_strings + 1 entries instead of one per byte."""
        from . import _lib
        from . import device as D

        alen = int(rbytes.numel())
        dev = rbytes.device
        own = getattr(self, "_recv", None)
        if own is not None and alen and own.data_ptr() == rbytes.data_ptr():
            arena = own  # received in place
        else:
            arena = D.alloc_arena(alen, dev)
            if alen:
                arena[:alen] = rbytes
        self._recv = None
        if alen == 0:
            starts = torch.zeros(0, dtype=torch.int64, device=dev)
            return D.DeviceStrings(arena, 0, starts), starts
        cap = (alen if n_strings is None else int(n_strings)) + 1
        handles = torch.empty(cap, dtype=torch.int64, device=dev)
        ws = torch.empty(16 + 4 * ((alen + 16383) // 16384), dtype=torch.uint8, device=dev)
        rank = torch.empty((alen + 63) // 64, dtype=torch.int32, device=dev)
        n = C.c_int64()
        _lib.check(_lib.lib().s5g_load_delimited_rank(arena.data_ptr(), alen, 0, handles.data_ptr(), cap,
                                                      C.byref(n), rank.data_ptr(), ws.data_ptr(),
                                                      ws.numel(),
                                                      torch.cuda.current_stream(dev).cuda_stream))
        starts = handles[: n.value]
        return D.DeviceStrings(arena, alen, starts, rank), starts

    def local_sort(self, ds, handles, want_lcps, **kw):
        """Sorted permutation of `handles` and the LCPs: s5g_sort, then
        s5g_input_positions (two stable radix sorts by handle: O(n), repeated
        handles allowed -- no per-arena-byte map)."""
        from . import device as D

        local = D.DeviceStrings(ds.arena, ds.arena_len, handles)
        out_h, lcps, _ = D.sort(local, want_lcps=want_lcps, **kw)
        self._sorted_h = out_h
        if ds.rank64 is not None and handles.data_ptr() == ds.handles.data_ptr():
            # the handles are the received arena's string starts: index by
            # the rank directory (s5g_rank_positions), no search and no sort
            return D.rank_positions(ds, out_h), lcps
        return D.input_positions(handles, out_h, ds.arena_len), lcps

    def sorted_handles(self, handles, perm):
        """handles[perm] -- the last local sort's own output when it is at hand."""
        out_h, self._sorted_h = getattr(self, "_sorted_h", None), None
        if out_h is not None and out_h.numel() == perm.numel():
            return out_h
        return self.take(handles, perm)

    def string_bytes(self, ds, h1: torch.Tensor) -> bytes:
        from . import device as D

        one = D.DeviceStrings(ds.arena, ds.arena_len, h1)
        L = int(D.lengths(one)[0].item())
        return ds.arena[int(h1[0]): int(h1[0]) + L].cpu().numpy().tobytes()
