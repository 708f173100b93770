"""Multi-rank S^5 (paper_1403_2056_b200.dist) on CPU: world_size 2 and 3 over
gloo, with an oracle-backed compute backend standing in for the GPU kernels.
Checks that the concatenation of the ranks' outputs is the reference's global
stable order and LCP array, including empty ranks, duplicates spanning ranks
and the replicated-arena (suffix) exchange mode."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1403_2056_b200 import corpora
from paper_1403_2056_b200.dist import (
    Shard,
    distributed_merge_sort,
    distributed_sort,
    handle_positions,
    pick_splitters,
    sample_positions,
)


class CpuBackend:
    """Test double: numpy / oracle implementations of the GPU compute steps."""

    comm_device = torch.device("cpu")

    def prepare(self, shard):
        return np.ascontiguousarray(shard.buffer, dtype=np.uint8)

    def _str(self, buf, h, maxlen=None):
        e = h
        while buf[e] != 0 and (maxlen is None or e - h < maxlen):
            e += 1
        return buf[h:e].tobytes()

    def sample(self, buf, shard, k, maxlen, seed=1, rank=0):
        pos = sample_positions(len(shard.handles), k, seed, rank)
        return [(self._str(buf, int(shard.handles[p]), maxlen), int(shard.base_index + p))
                for p in pos]

    def take(self, src, idx):
        return src[idx]

    def partition(self, buf, shard, sp, sp_g, handles=None, gidx=None):
        import bisect
        keys = list(zip(sp, sp_g))
        hs = shard.handles if handles is None else np.asarray(handles)
        gs = (shard.base_index + np.arange(len(hs))) if gidx is None else np.asarray(gidx)
        out = [bisect.bisect_right(keys, (self._str(buf, int(h)), int(g))) for h, g in zip(hs, gs)]
        return torch.tensor(out, dtype=torch.int32)

    def handles_of(self, buf, shard):
        return torch.from_numpy(np.asarray(shard.handles, dtype=np.int64))

    def sample_run(self, buf, handles, gidx, k, maxlen):
        n = len(handles)
        if n == 0:
            return []
        pos = np.unique(np.linspace(0, n - 1, num=min(k, n)).astype(np.int64))
        return [(self._str(buf, int(handles[p]), maxlen), int(gidx[p])) for p in pos]

    def fill_dchar(self, buf, sorted_h, lcps):
        return torch.from_numpy(oracle.fill_dchar(buf, sorted_h.numpy(), lcps.numpy()))

    def dest_counts(self, dest, G):
        return torch.bincount(dest.long(), minlength=G).tolist()

    def positions(self, buf, handles, query):
        return handle_positions(handles, query)

    def kway_merge(self, buf, run_off, handles, lcps, dchar):
        h, l, _ = oracle.kway_merge(buf, run_off, handles.numpy(), lcps.numpy(),
                                    dchar.numpy() if dchar is not None else None)
        return torch.from_numpy(h), torch.from_numpy(l)

    def group_by_dest(self, dest, G):
        order = torch.sort(dest, stable=True).indices
        return order, torch.bincount(dest.long(), minlength=G).tolist()

    def global_index(self, shard, order):
        return order.to(torch.int64) + shard.base_index

    def take_handles(self, buf, order):
        return torch.as_tensor(np.asarray(self._handles)[order.numpy()])

    def pack(self, buf, order, counts):
        h = self._handles[order.numpy()] if len(order) else np.zeros(0, np.int64)
        parts = [self._str(buf, int(x)) + b"\0" for x in h]
        bounds = np.r_[0, np.cumsum(counts)]
        byte_counts = [sum(len(p) for p in parts[bounds[q]:bounds[q + 1]]) for q in range(len(counts))]
        payload = torch.from_numpy(np.frombuffer(b"".join(parts), dtype=np.uint8).copy()) \
            if parts else torch.zeros(0, dtype=torch.uint8)
        return payload, byte_counts

    def unpack(self, rbytes):
        arr = rbytes.numpy().copy()
        zeros = np.flatnonzero(arr == 0)
        starts = np.r_[0, zeros[:-1] + 1].astype(np.int64) if len(zeros) else np.zeros(0, np.int64)
        return arr, torch.from_numpy(starts)

    def local_sort(self, buf, handles, want_lcps, **kw):
        h = handles.numpy()
        out, lcps, _ = oracle.s5_sort(buf, h)
        return handle_positions(handles, torch.from_numpy(out)), torch.from_numpy(lcps)

    def string_bytes(self, buf, h1):
        return self._str(buf, int(h1[0]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        buf, hnd, mode, cuts = case
        be = CpuBackend()
        lo, hi = cuts[rank], cuts[rank + 1]
        if mode in ("packed", "merge"):
            # each rank owns a self-contained buffer with its strings
            strs = [buf[h:buf.index(b"\0", h) + 1] for h in hnd[lo:hi]]
            sbuf = np.frombuffer(b"".join(strs), dtype=np.uint8).copy() if strs else np.zeros(0, np.uint8)
            shnd = np.r_[0, np.cumsum([len(x) for x in strs])[:-1]].astype(np.int64) if strs else np.zeros(0, np.int64)
        else:  # replicated arena: every rank holds the whole text
            sbuf = np.frombuffer(buf, dtype=np.uint8).copy()
            shnd = np.asarray(hnd[lo:hi], dtype=np.int64)
        be._handles = shnd
        if mode == "merge":
            res = distributed_merge_sort(Shard(sbuf, shnd, lo), be, samples_per_rank=16,
                                         max_splitter_len=6)
        else:
            res = distributed_sort(Shard(sbuf, shnd, lo), be, samples_per_rank=16,
                                   max_splitter_len=6, mode=mode)
        parts = [None] * world
        dist.all_gather_object(parts, (res.gidx.numpy(), res.lcps.numpy(), res.n_total))
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


def _run(world, buf, hnd, mode="packed", cuts=None):
    n = len(hnd)
    cuts = cuts or [(n * k) // world for k in range(world + 1)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (buf, hnd, mode, cuts), q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gidx = np.concatenate([p[0] for p in parts])
    lcps = np.concatenate([p[1] for p in parts])
    assert all(p[2] == n for p in parts)
    # oracle: global stable order and LCPs
    h, l, _ = oracle.s5_sort(np.frombuffer(buf, np.uint8), np.asarray(hnd, np.int64))
    want_gidx = handle_positions(torch.as_tensor(np.asarray(hnd, np.int64)), torch.from_numpy(h)).numpy()
    assert np.array_equal(gidx, want_gidx)
    assert np.array_equal(lcps, l)


def _pack(items):
    buf = b"".join(s + b"\0" for s in items)
    hnd = np.r_[0, np.cumsum([len(s) + 1 for s in items])[:-1]].astype(np.int64)
    return buf, hnd


def test_pick_splitters_is_order_statistics():
    s = [(b"b", 1), (b"a", 5), (b"a", 2), (b"c", 0)]
    sp, g = pick_splitters(s, 2)
    assert (sp, g) == ([b"b"], [1])


@pytest.mark.parametrize("world", [2, 3])
def test_random_strings(world):
    buf, hnd = corpora.gen_random(3000, 7)
    _run(world, buf.tobytes(), hnd)


def test_duplicates_across_ranks_keep_input_order():
    rng = np.random.default_rng(3)
    items = [bytes(rng.integers(97, 99, size=int(rng.integers(0, 4)), dtype=np.uint8)) for _ in range(1500)]
    buf, hnd = _pack(items)
    _run(2, buf, hnd)
    _run(3, buf, hnd)


def test_empty_rank_and_shared_prefixes():
    items = [b"http://same.host/" + bytes([97 + (i % 7)]) * (i % 5) for i in range(600)]
    buf, hnd = _pack(items)
    _run(3, buf, hnd, cuts=[0, 300, 300, 600])


def test_replicated_suffixes():
    buf, hnd = corpora.gen_suffix_markov(2000, chains=4)
    _run(2, buf.tobytes(), hnd, mode="replicated")


@pytest.mark.parametrize("world", [2, 3])
def test_merge_strategy_random(world):
    buf, hnd = corpora.gen_random(3000, 11)
    _run(world, buf.tobytes(), hnd, mode="merge")


def test_merge_strategy_duplicates_and_empty_rank():
    rng = np.random.default_rng(5)
    items = [bytes(rng.integers(97, 99, size=int(rng.integers(0, 4)), dtype=np.uint8)) for _ in range(1200)]
    buf, hnd = _pack(items)
    _run(2, buf, hnd, mode="merge")
    _run(3, buf, hnd, mode="merge", cuts=[0, 600, 600, 1200])


def test_merge_strategy_shared_prefixes():
    items = [b"http://same.host/" + bytes([97 + (i % 7)]) * (i % 5) for i in range(600)]
    buf, hnd = _pack(items)
    _run(3, buf, hnd, mode="merge")
