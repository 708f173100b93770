"""GPU K-way LCP merge (s5g_kway_merge; lcpmerge.py:25-424) and
partitioned_merge_sort (parallel.py:885-994) against the reference's own
merges (golden fixtures) and the oracle's loser tree."""

import numpy as np
import pytest

import golden_io as G
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_1403_2056_b200 as P  # noqa: E402
from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402


def _gpu_merge(buf, off, h, l, dchar=None, shared=0):
    ds = D.upload(buf, h)
    l_d = torch.from_numpy(np.ascontiguousarray(l, dtype=np.int64)).cuda()
    c_d = torch.from_numpy(np.ascontiguousarray(dchar, dtype=np.uint8)).cuda() if dchar is not None else None
    oh, ol = D.kway_merge(ds, off, ds.handles, l_d, c_d, shared)
    return oh.cpu().numpy(), ol.cpu().numpy()


@pytest.mark.parametrize("cached", [False, True])
@pytest.mark.parametrize("name", G.merges())
def test_kway_merge_matches_reference(name, cached):
    m = G.merge(name)
    c = G.case(m["case"])
    oh, ol = _gpu_merge(c["buffer"], m["run_off"], m["run_handles"], m["run_lcps"],
                        m["run_dchar"] if cached else None)
    assert np.array_equal(oh, m["out_handles"])
    assert ol[0] == 0
    assert np.array_equal(ol[1:], m["out_lcps"][1:])


def _runs(buf, handles, K, rng, empty_every=0):
    """Sort K random contiguous shards with the oracle; laid end to end
    (every empty_every-th shard empty when set)."""
    n = len(handles)
    cuts = np.r_[0, np.sort(rng.integers(0, n + 1, size=K - 1)), n].astype(np.int64)
    if empty_every:
        for j in range(1, K, empty_every):
            cuts[j + 1] = max(cuts[j + 1], cuts[j])
            cuts[j] = cuts[j + 1]  # shard j-1 absorbs, shard j is empty
        cuts = np.maximum.accumulate(cuts)
    hs, ls = [], []
    for j in range(K):
        sub = handles[cuts[j]:cuts[j + 1]]
        if len(sub):
            h, l, _ = oracle.parallel_s5(buf, sub)
        else:
            h, l = np.zeros(0, np.int64), np.zeros(0, np.int64)
        hs.append(h)
        ls.append(l)
    return cuts, np.concatenate(hs), np.concatenate(ls)


@pytest.mark.parametrize("K", [2, 3, 4, 7, 8, 16])
@pytest.mark.parametrize("gen", ["random", "dna", "urls", "suffixes"])
def test_kway_merge_random_shards_vs_oracle(K, gen):
    rng = np.random.default_rng(K * 31 + len(gen))
    buf, handles = {"random": lambda: corpora.gen_random(40_000, K),
                    "dna": lambda: corpora.gen_dna(30_000, 40, K),
                    "urls": lambda: corpora.gen_urls(30_000, K, hosts=200, pool=8),
                    "suffixes": lambda: corpora.gen_suffix_markov(20_000, K)}[gen]()
    off, h, l = _runs(buf, handles, K, rng, empty_every=3 if K >= 7 else 0)
    dchar = oracle.fill_dchar(buf, h, l)
    for cached in (False, True):
        oh, ol = _gpu_merge(buf, off, h, l, dchar if cached else None)
        eh, el, _ = oracle.kway_merge(buf, off, h, l, dchar if cached else None)
        assert np.array_equal(oh, eh)
        assert np.array_equal(ol, el)
        # and the merge of stable-sorted shards is the stable sort of the whole
        sh, sl, _ = oracle.parallel_s5(buf, handles)
        assert np.array_equal(oh, sh)
        assert np.array_equal(ol[1:], sl[1:])


def test_kway_merge_shared_prefix():
    c = G.case("depth3_900")
    rng = np.random.default_rng(3)
    off, h, l = _runs(c["buffer"], c["handles"], 4, rng)
    oh, ol = _gpu_merge(c["buffer"], off, h, l, None, shared=3)
    eh, el, _ = oracle.kway_merge(c["buffer"], off, h, l, None, 3)
    assert np.array_equal(oh, eh) and np.array_equal(ol, el)
    assert ol[0] == 3


def test_kway_merge_edge_cases():
    buf = b"b\0a\0b\0a\0\0"
    h = np.array([2, 0, 6, 4, 8], dtype=np.int64)  # "b","b" | "a"... as sorted runs below
    # runs: [a(6), b(0)] and [(empty)] and ["", a(2)?] -- build from the oracle
    runs = [np.array([6, 0], np.int64), np.zeros(0, np.int64), np.array([8, 4, 2], np.int64)]
    hs, ls = [], []
    for r in runs:
        if len(r):
            sh, sl, _ = oracle.parallel_s5(buf, r)
        else:
            sh, sl = r, r
        hs.append(sh), ls.append(sl)
    off = np.r_[0, np.cumsum([len(x) for x in hs])]
    oh, ol = _gpu_merge(buf, off, np.concatenate(hs), np.concatenate(ls))
    eh, el, _ = oracle.kway_merge(buf, off, np.concatenate(hs), np.concatenate(ls))
    assert np.array_equal(oh, eh) and np.array_equal(ol, el)
    # one run: a copy; zero strings: nothing
    oh, ol = _gpu_merge(buf, np.array([0, 2]), hs[0], ls[0])
    assert np.array_equal(oh, hs[0]) and ol[0] == 0
    with pytest.raises(ValueError):
        _gpu_merge(buf, np.arange(18), np.zeros(17, np.int64), np.zeros(17, np.int64))


def test_lcpmerge_api_mirrors_reference():
    m = G.merge("merge_urls_2000_k3")
    c = G.case(m["case"])
    s = P.StringSet(c["buffer_bytes"], c["handles"])
    off = m["run_off"]
    streams = [P.LcpStream(s, m["run_handles"][off[j]:off[j + 1]], m["run_lcps"][off[j]:off[j + 1]],
                           m["run_dchar"][off[j]:off[j + 1]]) for j in range(len(off) - 1)]
    for cached in (False, True):
        h, l = P.kway_lcp_merge(streams, cached=cached)
        assert np.array_equal(h, m["out_handles"]) and np.array_equal(l, m["out_lcps"])
    h, l = P.binary_lcp_merge(streams[0], streams[1])
    n2 = off[2]
    eh, el, _ = oracle.kway_merge(c["buffer"], off[:3], m["run_handles"][:n2], m["run_lcps"][:n2])
    assert np.array_equal(h, eh) and l[0] == -1 and np.array_equal(l[1:], el[1:])


@pytest.mark.parametrize("K", [1, 2, 4, 8, 16, 17, 40])
@pytest.mark.parametrize("name", ["random_3000", "urls_2000", "dups_2000", "deep_prefix_1500",
                                  "suffixes_1800", "all_equal_700", "shuffled_dups_2500",
                                  "random_n17", "random_n2"])
def test_partitioned_merge_sort_golden(name, K):
    c = G.case(name)
    s = P.StringSet(c["buffer_bytes"], c["handles"])
    res = P.partitioned_merge_sort(s, K=K, want_lcps=True)
    assert np.array_equal(res.set.handles, c["out_handles"])
    assert np.array_equal(res.lcps, c["lcps"])
    out = P.partitioned_merge_sort(s, K=K, use_cache=False)
    assert np.array_equal(out.handles, c["out_handles"])


@pytest.mark.parametrize("cfg,scale", [("c1_random", 1.0), ("c2_dna", 1 / 16), ("c3_urls", 1 / 8),
                                       ("c4_suffixes", 1 / 16)])
def test_partitioned_merge_sort_scaled_configs(cfg, scale):
    buf, handles = corpora.CONFIGS[cfg](scale)
    s = P.StringSet(buf.tobytes(), handles)
    res = P.partitioned_merge_sort(s, K=8, want_lcps=True)
    status, bad = oracle.certify(buf, handles, res.set.handles, res.lcps)
    assert status == 0, (oracle.CERT_STATUS[status], bad)


def test_kway_lcp_merge_more_than_16_streams():
    """K > 16 (the reference takes any K): merged in rounds of 16-run groups."""
    c = G.case("random_3000")
    s = P.StringSet(c["buffer_bytes"], c["handles"])
    K = 37
    cuts = np.linspace(0, len(c["handles"]), K + 1).astype(np.int64)
    hs, ls = [], []
    for j in range(K):
        r = P.s5_sort(s.with_handles(c["handles"][cuts[j]:cuts[j + 1]]), want_lcps=True)
        hs.append(r.set.handles)
        ls.append(r.lcps)
    H, L = np.concatenate(hs), np.concatenate(ls)
    streams = [P.LcpStream(s, H, L, None, int(cuts[j]), int(cuts[j + 1] - cuts[j])) for j in range(K)]
    for cached in (False, True):
        oh, ol = P.kway_lcp_merge(streams, cached=cached)
        assert np.array_equal(oh, c["out_handles"])
        assert np.array_equal(ol[1:], c["lcps"][1:]) and ol[0] == -1
