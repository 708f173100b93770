"""GPU forms of the input side (load_delimited, strset.py:113-134) and of
dist_stats (strset.py:290-309), against the host mirror / the oracle."""

import numpy as np
import pytest

import golden_io as G
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402
from paper_1403_2056_b200 import load_delimited  # noqa: E402


@pytest.mark.parametrize("name", sorted(G.load_cases()))
def test_load_delimited_matches_reference_golden(name):
    """GPU load_delimited against the reference's own outputs
    (tests/golden/golden_load.npz, made by make_golden_load.py from
    strsort.strset.load_delimited, strset.py:113-134)."""
    c = G.load_cases()[name]
    data = c["input"].tobytes()
    if c["error"]:
        with pytest.raises(ValueError, match="reserved as terminator"):
            D.load_delimited(data, c["delimiter"])
        with pytest.raises(ValueError, match="reserved as terminator"):
            load_delimited(data, c["delimiter"])
        return
    ds = D.load_delimited(data, c["delimiter"])
    assert ds.arena_len == len(c["buffer"])
    assert np.array_equal(ds.arena[: ds.arena_len].cpu().numpy(), c["buffer"])
    assert np.array_equal(ds.handles.cpu().numpy(), c["handles"])
    s = load_delimited(data, c["delimiter"])  # the package-level (GPU) entry
    assert s.buffer == c["buffer"].tobytes() and np.array_equal(s.handles, c["handles"])


def test_load_delimited_large_then_sort():
    rng = np.random.default_rng(0)
    lines = [bytes(rng.integers(97, 123, size=int(rng.integers(0, 30)), dtype=np.uint8))
             for _ in range(200_000)]
    raw = b"\n".join(lines)
    ds = D.load_delimited(raw, 10)
    buf = raw.replace(b"\n", b"\0") + b"\0"
    starts = np.concatenate(([0], np.flatnonzero(np.frombuffer(buf, np.uint8) == 0)[:-1] + 1))
    assert np.array_equal(ds.handles.cpu().numpy(), starts)
    h, l, _ = D.sort(ds, want_lcps=True)
    oh, ol, _ = oracle.parallel_s5(buf, starts)
    assert np.array_equal(h.cpu().numpy(), oh) and np.array_equal(l.cpu().numpy(), ol)


@pytest.mark.parametrize("name", ["random_3000", "dups_2000", "all_equal_700", "urls_2000"])
def test_dist_stats_matches_golden(name):
    c = G.case(name)
    lcps = torch.from_numpy(c["lcps"]).cuda()
    assert D.dist_stats(lcps) == (c["D"], c["L"])


def test_dist_stats_full_c2():
    buf, hnd = corpora.gen_dna(1 << 20)
    ds = D.upload(buf, hnd)
    h, l, _ = D.sort(ds, want_lcps=True)
    oh, ol, _ = oracle.parallel_s5(buf, hnd)
    D_, L_, _ = oracle.dist_stats(buf, oh, ol)
    assert D.dist_stats(l) == (D_, L_)


def _received(raw: bytes):
    """A received payload (strings back to back, each with its terminator)
    loaded the way the multi-GPU path does (GpuBackend.recv_arena + unpack)."""
    from paper_1403_2056_b200.dist import GpuBackend

    be = GpuBackend()
    view = be.recv_arena(len(raw))
    view.copy_(torch.from_numpy(np.frombuffer(raw, np.uint8).copy()))
    return be, view


@pytest.mark.parametrize("seed,maxlen", [(0, 0), (1, 5), (2, 70), (3, 300)])
def test_rank_directory_positions(seed, maxlen):
    """s5g_load_delimited_rank + s5g_rank_positions: every string start maps
    back to its index (empty strings, strings spanning several 64-byte blocks,
    several starts inside one block), in any query order; the starts equal the
    plain load_delimited's."""
    rng = np.random.default_rng(seed)
    strs = [bytes(rng.integers(1, 256, size=int(rng.integers(0, maxlen + 1)), dtype=np.uint8))
            for _ in range(5000)]
    raw = b"".join(s + b"\0" for s in strs)
    be, view = _received(raw)
    ds, starts = be.unpack(view, len(strs))
    assert ds.arena.data_ptr() == view.data_ptr()  # adopted in place, no copy
    want = np.concatenate(([0], np.cumsum([len(s) + 1 for s in strs])[:-1]))
    assert np.array_equal(starts.cpu().numpy(), want)
    perm = torch.from_numpy(rng.permutation(len(strs))).cuda()
    pos = D.rank_positions(ds, starts[perm])
    assert torch.equal(pos, perm)
    assert torch.equal(D.input_positions(starts, starts[perm], ds.arena_len), perm)  # ascending fast path


def test_load_delimited_n_capacity():
    """A receiver that under-states the string count gets an error, not an
    overrun of its starts buffer."""
    raw = b"ab\0c\0\0dd\0"
    be, view = _received(raw)
    with pytest.raises(ValueError, match="room"):
        be.unpack(view, 2)
    be, view = _received(raw)
    ds, starts = be.unpack(view, 4)
    assert starts.cpu().tolist() == [0, 3, 5, 6]


def test_pack_order_lane_groups():
    """s5g_pack_plan + s5g_pack (eight lanes per string, four strings per
    group): strings of every length around the 8-byte and 64-byte round
    boundaries, at every source and destination alignment."""
    rng = np.random.default_rng(5)
    lens = list(range(0, 200)) + [255, 256, 257, 511, 512, 513, 1000]
    strs = [bytes(rng.integers(1, 256, size=L, dtype=np.uint8)) for L in lens for _ in range(3)]
    rng.shuffle(strs)
    buf = b"".join(s + b"\0" for s in strs)
    hnd = np.concatenate(([0], np.cumsum([len(s) + 1 for s in strs])[:-1])).astype(np.int64)
    ds = D.upload(buf, hnd)
    order = torch.from_numpy(rng.permutation(len(strs))).cuda()
    payload, dest_bytes = D.pack_order(ds, order, [100, len(strs) - 100])
    o = order.cpu().numpy()
    want = b"".join(strs[i] + b"\0" for i in o)
    assert payload.cpu().numpy().tobytes() == want
    assert dest_bytes == [sum(len(strs[i]) + 1 for i in o[:100]), sum(len(strs[i]) + 1 for i in o[100:])]
