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
from paper_1403_2056_b200.strset import load_delimited  # noqa: E402


@pytest.mark.parametrize("data,delim", [
    (b"a\0b\0", 0), (b"ab\ncd\n", 10), (b"ab\ncd", 10), (b"", 10), (b"\n\n", 10),
    (b"x", 0), (b"abc\0\0d", 0)])
def test_load_delimited_matches_host(data, delim):
    want = load_delimited(data, delim)
    ds = D.load_delimited(data, delim)
    assert ds.arena_len == len(want.buffer)
    assert bytes(ds.arena[: ds.arena_len].cpu().numpy()) == want.buffer
    assert np.array_equal(ds.handles.cpu().numpy(), want.handles)


def test_load_delimited_rejects_zero_with_delimiter():
    with pytest.raises(ValueError, match="reserved as terminator"):
        D.load_delimited(b"a\0b\n", 10)


def test_load_delimited_large_then_sort():
    rng = np.random.default_rng(0)
    lines = [bytes(rng.integers(97, 123, size=int(rng.integers(0, 30)), dtype=np.uint8))
             for _ in range(200_000)]
    raw = b"\n".join(lines)
    want = load_delimited(raw, 10)
    ds = D.load_delimited(raw, 10)
    assert np.array_equal(ds.handles.cpu().numpy(), want.handles)
    h, l, _ = D.sort(ds, want_lcps=True)
    oh, ol, _ = oracle.parallel_s5(want.buffer, want.handles)
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
