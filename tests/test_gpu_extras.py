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
