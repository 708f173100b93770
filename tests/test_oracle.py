"""Pin the CPU oracle (oracle/s5_oracle.c) against the reference's own outputs.

The golden vectors were produced by running the reference (strsort 0.1.0)
with tests/golden/make_golden.py.  Every function of the restatement that the
parity tests rely on is checked here: extract_keys, select_splitters,
classify (both variants), distribute, s5_sort, parallel_s5, mkqs_cached,
lcp_insertion_sort, lcp_array_oracle, dist_stats, fill_dchar and the K11
certificate.
"""

import numpy as np
import pytest

import oracle
import golden_io as G

CASES = G.cases()
KATS = G.kats()


@pytest.mark.parametrize("name", CASES)
def test_s5_sort_matches_reference(name):
    c = G.case(name)
    for kw in ({}, {"t_medium": 16}, {"t_medium": 200, "variant": "equal"}, {"v": 7, "t_medium": 32}):
        h, lcps, _ = oracle.s5_sort(c["buffer_bytes"], c["handles"], depth=c["depth"], **kw)
        assert np.array_equal(h, c["out_handles"]), kw
        assert np.array_equal(lcps, c["lcps"]), kw
    assert np.array_equal(oracle.fill_dchar(c["buffer_bytes"], h, lcps), c["dchar"])


@pytest.mark.parametrize("name", [n for n in CASES if G.case(n)["depth"] == 0])
@pytest.mark.parametrize("p", [1, 2, 4])
def test_parallel_s5_matches_reference(name, p):
    c = G.case(name)
    h, lcps, _ = oracle.parallel_s5(c["buffer_bytes"], c["handles"], p=p, t_medium=128)
    assert np.array_equal(h, c["out_handles"])
    assert np.array_equal(lcps, c["lcps"])


@pytest.mark.parametrize("name", [n for n in CASES if G.case(n)["depth"] == 0])
def test_mkqs_and_keys_and_stats(name):
    c = G.case(name)
    buf = c["buffer_bytes"]
    h, lcps, st = oracle.mkqs_cached(buf, c["handles"])
    assert np.array_equal(h, c["mkqs_handles"])
    assert np.array_equal(lcps[1:], c["lcps"][1:])
    assert st["word_fetches"] == c["mkqs_word_fetches"]
    for dep in (0, 2, 5, 9):
        assert np.array_equal(oracle.extract_keys(buf, c["handles"], dep), c[f"keys_d{dep}"])
    if "ins_handles" in c:
        h2, l2, st2 = oracle.lcp_insertion_sort(buf, c["handles"])
        assert np.array_equal(h2, c["ins_handles"])
        assert np.array_equal(l2, c["ins_lcps"])
        assert st2["char_cmps"] == c["ins_char_cmps"]
    if c["n"]:
        D, L, _ = oracle.dist_stats(buf, c["out_handles"], c["lcps"])
        assert (D, L) == (c["D"], c["L"])
        assert np.array_equal(oracle.lcp_array(buf, c["out_handles"]), c["lcps"])
    assert oracle.certify(buf, c["handles"], c["out_handles"], c["lcps"]) == (0, -1)


@pytest.mark.parametrize("name", KATS)
def test_splitters_classify_distribute(name):
    k = G.kat(name)
    t = oracle.select_splitters(k["sample"], k["v"])
    for fld in ("tree", "inorder", "node_to_inorder", "slcp", "eq_leftmost", "term_pos"):
        assert np.array_equal(getattr(t, fld), k[fld]), fld
    assert np.array_equal(t.eq_final, k["eq_final"].astype(bool))
    for variant in ("unroll", "equal"):
        assert np.array_equal(oracle.classify_keys(k["keys"], t, variant), k["oracle"])
    out, bounds = oracle.distribute(np.arange(len(k["keys"])) * 3, k["oracle"], 2 * k["v"] + 1)
    assert np.array_equal(out, k["dist_handles"])
    assert np.array_equal(bounds, k["dist_bounds"])


def word(b: bytes) -> int:
    return int.from_bytes((b + b"\0" * 8)[:8], "big")


def test_reference_known_answers():
    # test_ssss.py:55-98 / test_strset.py:53-172 known answers, restated
    sample = np.array([word(bytes([c])) for c in range(65, 74)], dtype=np.uint64)
    t = oracle.select_splitters(sample, 3)
    assert list(t.inorder) == [sample[2], sample[4], sample[7]]
    t = oracle.select_splitters(np.full(9, word(b"same"), np.uint64), 3)
    assert t.eq_final.all()
    s = np.array(sorted([word(b"abcx"), word(b"abcy"), word(b"q")] * 3), np.uint64)
    assert list(oracle.select_splitters(s, 3).slcp) == [0, 3, 0, 0]
    t = oracle.select_splitters(np.full(3, word(b"m"), np.uint64), 1)
    keys = np.array([word(b"a"), word(b"m"), word(b"z")], np.uint64)
    assert list(oracle.classify_keys(keys, t)) == [0, 1, 2]
    out, bounds = oracle.distribute(np.array([10, 20, 30]), np.array([1, 0, 1]), 3)
    assert list(bounds) == [0, 1, 3, 3] and list(out) == [20, 10, 30]
    assert oracle.shared_chars(word(b"abcdefgh"), word(b"abcxefgh")) == 3
    assert oracle.shared_chars(word(b"ab"), word(b"ab")) == 2
    assert oracle.shared_chars(word(b"abcdefgh"), word(b"abcdefgh")) == 8
    buf = b"ab\0cd\0"
    assert oracle.extract_keys(buf, [0], 0)[0] == word(b"ab")
    assert oracle.extract_keys(b"\0x\0", [0], 5)[0] == 0
    assert oracle.tree_capacity(10**6) == 8191 and oracle.tree_capacity(10) == 3


def test_certificate_detects_faults():
    c = G.case("dups_2000")
    buf, hin, hout, lcps = c["buffer_bytes"], c["handles"], c["out_handles"], c["lcps"]
    assert oracle.certify(buf, hin, hout, lcps)[0] == 0
    bad = hout.copy(); bad[5] = bad[6]
    assert oracle.certify(buf, hin, bad, lcps)[0] == 1
    bad = hout.copy(); bad[[10, 1500]] = bad[[1500, 10]]
    assert oracle.certify(buf, hin, bad, None)[0] == 2
    # swap two equal strings: stability violation
    s = [buf[h:buf.index(b"\0", h)] for h in hout]
    i = next(i for i in range(1, len(s)) if s[i] == s[i - 1])
    bad = hout.copy(); bad[[i - 1, i]] = bad[[i, i - 1]]
    assert oracle.certify(buf, hin, bad, lcps)[0] == 3
    badl = lcps.copy(); badl[7] += 1
    assert oracle.certify(buf, hin, hout, badl)[0] == 4


# --- K-way LCP merge (lcpmerge.py) against the reference's own merges --------

@pytest.mark.parametrize("name", G.merges())
@pytest.mark.parametrize("cached", [False, True])
def test_oracle_kway_merge_matches_reference(name, cached):
    m = G.merge(name)
    c = G.case(m["case"])
    oh, ol, st = oracle.kway_merge(c["buffer"], m["run_off"], m["run_handles"], m["run_lcps"],
                                   m["run_dchar"] if cached else None)
    ol[0] = -1  # the reference's LCP_UNDEF convention without output arrays
    assert np.array_equal(oh, m["out_handles"])
    assert np.array_equal(ol, m["out_lcps"])
    if cached:
        _, _, st0 = oracle.kway_merge(c["buffer"], m["run_off"], m["run_handles"], m["run_lcps"])
        assert st["merge_buffer_cmps"] <= st0["merge_buffer_cmps"]
