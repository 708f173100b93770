"""Host-side logic of the drop-in (no GPU): argument errors, data model,
splitter-tree metadata for step hooks, corpora."""

import numpy as np
import pytest

import oracle
import golden_io as G
from paper_1403_2056_b200 import corpora
from paper_1403_2056_b200.ssss import SplitterTree, check_set, s5_sort, tree_capacity
from paper_1403_2056_b200.strset import (
    StringSet, from_strings, shared_chars, word_terminator_pos)


def test_unknown_variant_is_value_error():
    s = from_strings([b"a", b"b"])
    with pytest.raises(ValueError, match="unknown classify variant"):
        s5_sort(s, variant="bogus")


def test_not_zero_terminated():
    with pytest.raises(ValueError, match="not zero-terminated"):
        check_set(b"abc", np.array([0]))
    with pytest.raises(ValueError, match="not zero-terminated"):
        check_set(b"ab\0cd", np.array([0, 3]))
    check_set(b"ab\0cd", np.array([0]))
    check_set(b"", np.zeros(0, np.int64))


def test_empty_set_needs_no_device():
    res = s5_sort(from_strings([]), want_lcps=True, want_dchar=True)
    assert len(res.set) == 0 and len(res.lcps) == 0 and len(res.dchar) == 0


def test_from_strings():
    s = from_strings([b"x", b"", b"yz"])
    assert s.buffer == b"x\0\0yz\0" and list(s.handles) == [0, 2, 3]
    assert from_strings([]).buffer == b"" and len(from_strings([]).handles) == 0
    with pytest.raises(ValueError, match="terminator"):
        from_strings([b"a\0b"])


def test_load_delimited_golden_fixtures_are_consistent():
    """tests/golden/golden_load.npz holds the reference's own load_delimited
    outputs (make_golden_load.py); the GPU path is checked against them in
    test_gpu_extras.py.  Here: every fixture is a well-formed string set."""
    for name, c in G.load_cases().items():
        if c["error"]:
            assert 0 in c["input"] and c["delimiter"] != 0
            continue
        buf, h = c["buffer"], c["handles"]
        assert len(buf) == 0 or buf[-1] == 0
        assert (len(h) == 0 and len(buf) == 0) or (h[0] == 0 and (buf[h[1:] - 1] == 0).all())
        assert int((buf == 0).sum()) == len(h)


@pytest.mark.parametrize("name", G.kats())
def test_splitter_tree_metadata_matches_reference(name):
    k = G.kat(name)
    t = SplitterTree.from_inorder(k["v"], k["inorder"])
    for fld in ("tree", "node_to_inorder", "slcp", "eq_leftmost", "term_pos"):
        assert np.array_equal(getattr(t, fld), k[fld]), fld
    assert np.array_equal(t.eq_final, k["eq_final"].astype(bool))


def test_word_helpers_match_oracle():
    rng = np.random.default_rng(0)
    a = rng.integers(0, 4, size=(500, 8), dtype=np.uint8)
    b = a.copy(); b[:, 5] ^= rng.integers(0, 2, size=500, dtype=np.uint8)
    ka = a.view(">u8").reshape(-1).astype(np.uint64)
    kb = b.view(">u8").reshape(-1).astype(np.uint64)
    assert list(word_terminator_pos(ka)) == [oracle.term_pos(x) for x in ka]
    assert list(shared_chars(ka, kb)) == [oracle.shared_chars(x, y) for x, y in zip(ka, kb)]


def test_tree_capacity_matches_oracle():
    for n in (0, 1, 2, 3, 5, 16, 100, 16381, 16382, 10**7):
        for v in (1, 7, 8191, 10000):
            assert tree_capacity(n, v) == oracle.tree_capacity(n, v)


def test_corpora_shapes():
    buf, h = corpora.gen_dna(1000)
    assert len(h) == 1000 and buf[100] == 0 and set(np.unique(buf[:100])) <= set(b"ACGT")
    buf, h = corpora.gen_suffix_markov(1 << 14, chains=16)
    assert len(h) == 1 << 14 and buf[-1] == 0 and (buf[:-1] >= 97).all()
    buf, h = corpora.gen_urls(2000, hosts=50, pool=8)
    s = StringSet(buf.tobytes(), h)
    assert all(x.startswith(b"http://") for x in s.strings()[:50])
    buf, h = corpora.gen_nodup(5000)
    s = StringSet(buf.tobytes(), h)
    strs = s.strings()
    assert len(set(strs)) == 5000 and all(32 <= len(x) <= 200 for x in strs)


def test_nodup_generator_definition():
    """C5 generator (csrc/s5g_gen.cu): counter-based, so a smaller corpus is a
    prefix of a larger one; lengths U[32,200]; a base-36 counter suffix; the
    16-character prefix is one of at most 2^16 vocabulary words."""
    n = 20000
    buf, h = corpora.gen_nodup(n)
    assert len(buf) == corpora.nodup_bytes(n) and h[0] == 0
    b2, h2 = corpora.gen_nodup(n // 3)
    assert np.array_equal(h2, h[: n // 3]) and np.array_equal(b2, buf[: len(b2)])
    strs = StringSet(buf.tobytes(), h).strings()
    lens = np.array([len(x) for x in strs])
    assert lens.min() == 32 and lens.max() == 200 and abs(lens.mean() - 116) < 2
    for i in (0, 1, 35, 36, 12345, n - 1):
        assert int(strs[i][-6:].decode(), 36) == i
    assert all(x[:-6].isalpha() and x.islower() for x in strs[:500])
    prefixes = {x[:16] for x in strs}
    assert len(prefixes) <= 1 << 16 and len(prefixes) > n * 0.8  # 2^16 words, n << 2^16 draws
    assert len(set(strs)) == n
    assert corpora.gen_nodup(1000, seed=5)[0][:64].tobytes() != buf[:64].tobytes()


def test_register_with_reference_harness():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import strsort.bench as B
    except ImportError:
        pytest.skip("reference not importable here")
    from paper_1403_2056_b200.bench_api import register_with_strsort
    assert register_with_strsort()
    assert "gpu-s5" in B.ALGORITHMS and "gpu-ps5" in B.ALGORITHMS


def test_parallel_s5_p_beyond_visible_devices_is_a_value_error():
    """p counts GPUs (parallel.py:468-492's p counts workers); more than the
    visible devices is refused before any device work."""
    import paper_1403_2056_b200 as P
    s = from_strings([b"b", b"a"])
    with pytest.raises(ValueError, match="exceeds"):
        P.parallel_s5(s, p=P.parallel.visible_devices() + 1)
    with pytest.raises(ValueError, match="unknown classify variant"):
        P.parallel_s5(s, p=1, variant="bogus")
