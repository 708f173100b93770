"""GPU pieces of the multi-GPU path: the partition / lengths / pack kernels
against the CPU test backend, and a world_size-1 NCCL run of the whole
distributed sort (the exchange degenerates, every kernel still runs)."""

import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402
from paper_1403_2056_b200.dist import (GpuBackend, Shard, distributed_merge_sort,  # noqa: E402
                                       distributed_sort, handle_positions, pick_splitters)
from test_dist import CpuBackend  # noqa: E402


def test_partition_lengths_pack_match_cpu_backend():
    buf, hnd = corpora.gen_urls(5000, hosts=40, pool=6)
    shard = Shard(buf, hnd, 777)
    cpu, gpu = CpuBackend(), GpuBackend()
    cpu._handles = hnd
    ds = gpu.prepare(shard)
    samples = cpu.sample(buf, shard, 64, 12)
    for G in (2, 3, 8):
        sp, g = pick_splitters(samples, G)
        assert np.array_equal(gpu.partition(ds, shard, sp, g).cpu().numpy(),
                              cpu.partition(buf, shard, sp, g).numpy())
    assert np.array_equal(D.lengths(ds).cpu().numpy(), oracle.lengths(buf, hnd))
    dest = gpu.partition(ds, shard, *pick_splitters(samples, 4))
    order, counts = gpu.group_by_dest(dest, 4)
    payload, bc = gpu.pack(ds, order, counts)
    p2, bc2 = cpu.pack(buf, order.cpu(), counts)
    assert bc == bc2 and np.array_equal(payload.cpu().numpy(), p2.numpy())


def test_distributed_sort_world1_nccl():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        for cfg in ("c1_random", "c3_urls"):
            buf, hnd = corpora.CONFIGS[cfg](1 / 64)
            h, l, _ = oracle.parallel_s5(buf, hnd)
            want = handle_positions(torch.from_numpy(hnd), torch.from_numpy(h)).numpy()
            for strategy in (distributed_sort, distributed_merge_sort):
                res = strategy(Shard(buf, hnd, 0), GpuBackend(), samples_per_rank=64)
                assert np.array_equal(res.gidx.cpu().numpy(), want), strategy.__name__
                assert np.array_equal(res.lcps.cpu().numpy(), l), strategy.__name__
    finally:
        dist.destroy_process_group()


def test_merge_strategy_pieces_match_cpu_backend():
    """sample_run / partition on a sorted run / fill_dchar / kway_merge of the
    GPU backend equal the CPU test backend's."""
    buf, hnd = corpora.gen_dna(20_000, 30, 5)
    shard = Shard(buf, hnd, 123)
    cpu, gpu = CpuBackend(), GpuBackend()
    cpu._handles = hnd
    ds = gpu.prepare(shard)
    perm, lcps = gpu.local_sort(ds, ds.handles, True)
    sh = ds.handles[perm]
    gidx = perm + 123
    s_gpu = gpu.sample_run(ds, sh, gidx, 50, 10)
    s_cpu = cpu.sample_run(buf, sh.cpu().numpy(), gidx.cpu().numpy(), 50, 10)
    assert s_gpu == s_cpu
    sp, g = pick_splitters(s_gpu * 3, 4)
    d_gpu = gpu.partition(ds, shard, sp, g, handles=sh, gidx=gidx).cpu().numpy()
    d_cpu = cpu.partition(buf, shard, sp, g, handles=sh.cpu().numpy(), gidx=gidx.cpu().numpy()).numpy()
    assert np.array_equal(d_gpu, d_cpu) and np.all(np.diff(d_gpu) >= 0)
    dc = gpu.fill_dchar(ds, sh, lcps).cpu().numpy()
    assert np.array_equal(dc, cpu.fill_dchar(buf, sh.cpu(), lcps.cpu()).numpy())


@pytest.mark.parametrize("G", [1, 2, 7, 64, 127])
@pytest.mark.parametrize("n", [1, 2047, 2048, 2049, 100_000])
def test_group_by_dest_is_stable_counting_sort(n, G):
    rng = np.random.default_rng(n + G)
    dest = torch.from_numpy(rng.integers(0, G, size=n).astype(np.int32)).cuda()
    order, counts = D.group_by_dest(dest, G)
    want = torch.sort(dest.cpu().long(), stable=True).indices  # test-side reference
    assert torch.equal(order.cpu(), want)
    assert counts.cpu().tolist() == torch.bincount(dest.cpu().long(), minlength=G).tolist()


def test_positions_inverts_unique_handles():
    rng = np.random.default_rng(9)
    h = torch.from_numpy(rng.permutation(1 << 20)[:300_000].astype(np.int64)).cuda()
    q = h[torch.from_numpy(rng.permutation(300_000)).cuda()]
    pos = D.positions(h, q, 1 << 20)
    assert torch.equal(h[pos], q)
    assert torch.equal(pos.cpu(), handle_positions(h.cpu(), q.cpu()))


@pytest.mark.parametrize("n,dups", [(1, False), (1000, False), (200_000, False), (50_000, True)])
def test_input_positions_with_repeated_handles(n, dups):
    """s5g_input_positions: the input position of every output string of a
    stable sort, repeated handles (the same string) matched in input order --
    what local_sort needs without an arena-sized map."""
    rng = np.random.default_rng(n)
    items = [bytes(rng.integers(97, 100, size=int(rng.integers(0, 6)), dtype=np.uint8))
             for _ in range(max(1, n // 4 if dups else n))]
    buf = b"".join(x + b"\0" for x in items)
    starts = np.concatenate(([0], np.cumsum([len(x) + 1 for x in items])[:-1])).astype(np.int64)
    hnd = rng.choice(starts, size=n) if dups else rng.permutation(starts)[:n]
    ds = D.upload(buf, hnd)
    out_h, _, _ = D.sort(ds, want_lcps=False)
    pos = D.input_positions(ds.handles, out_h, ds.arena_len).cpu().numpy()
    assert np.array_equal(np.sort(pos), np.arange(n))          # a permutation
    assert np.array_equal(hnd[pos], out_h.cpu().numpy())       # of the right strings
    oh, _, _ = oracle.parallel_s5(buf, hnd)
    # stable: equal strings keep input order -> the oracle's order of positions
    want = np.argsort(np.array([buf[h:buf.index(b"\0", h)] for h in hnd], dtype=object), kind="stable")
    assert np.array_equal(pos, want)


def test_pack_order_matches_host_packing():
    buf, hnd = corpora.gen_urls(5000, 3)
    ds = D.upload(buf, hnd)
    order = torch.as_tensor(np.random.default_rng(1).permutation(len(hnd)), device="cuda")
    counts = [1200, 0, 3800]
    payload, bc = D.pack_order(ds, order, counts)
    o = order.cpu().numpy()
    parts = [buf[h:np.flatnonzero(buf[h:] == 0)[0] + h].tobytes() + b"\0" for h in hnd[o]]
    assert payload.cpu().numpy().tobytes() == b"".join(parts)
    assert bc == [sum(len(p) for p in parts[:1200]), 0, sum(len(p) for p in parts[1200:])]
