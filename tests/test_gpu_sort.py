"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the pinned CPU oracle.  Bit-exact handles, LCPs, dchar."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import golden_io as G
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_1403_2056_b200 as P  # noqa: E402
from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


KWS = [{}, {"t_medium": 16}, {"t_medium": 200, "variant": "equal"}, {"v": 7, "t_medium": 40},
       {"seed": 5, "t_medium": 1000}]


@pytest.mark.parametrize("kw", KWS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "default")
@pytest.mark.parametrize("name", G.cases())
def test_golden_parity(name, kw):
    c = G.case(name)
    s = P.StringSet(c["buffer_bytes"], c["handles"])
    res = P.s5_sort(s, depth=c["depth"], want_lcps=True, want_dchar=True, **kw)
    assert np.array_equal(res.set.handles, c["out_handles"])
    assert np.array_equal(res.lcps, c["lcps"])
    assert np.array_equal(res.dchar, c["dchar"])


def test_return_types_follow_reference():
    c = G.case("random_3000")
    s = P.StringSet(c["buffer_bytes"], c["handles"])
    out = P.s5_sort(s)
    assert isinstance(out, P.StringSet) and np.array_equal(out.handles, c["out_handles"])
    out = P.s5_sort(s, want_dchar=True)  # reference: dchar without lcps -> StringSet
    assert isinstance(out, P.StringSet)
    stats = P.SortStats()
    res = P.parallel_s5(s, p=1, want_dchar=True, stats=stats)
    assert np.array_equal(res.lcps, c["lcps"]) and np.array_equal(res.dchar, c["dchar"])
    assert stats.scratch_words == 3000 and stats.word_fetches >= 3000
    assert np.array_equal(s.handles, c["handles"])  # input never mutated


text = st.binary(min_size=0, max_size=24).map(lambda b: bytes(c if c else 1 for c in b))


@given(st.lists(text, max_size=300), st.sampled_from([16, 64, 1 << 20]),
       st.sampled_from(["unroll", "equal"]))
@settings(max_examples=60, deadline=None)
def test_property_vs_oracle(items, t_medium, variant):
    s = P.from_strings(items)
    res = P.s5_sort(s, want_lcps=True, t_medium=t_medium, variant=variant)
    h, lcps, _ = oracle.s5_sort(s.buffer, s.handles)
    assert np.array_equal(res.set.handles, h)
    assert np.array_equal(res.lcps, lcps)


def test_kernel_extract_keys():
    for name in ("random_3000", "high_bytes_1500", "all_empty_300", "suffixes_1800"):
        c = G.case(name)
        ds = D.upload(c["buffer_bytes"], c["handles"])
        for dep in (0, 2, 5, 9):
            got = D.extract_keys(ds, dep).cpu().numpy().view(np.uint64)
            assert np.array_equal(got, c[f"keys_d{dep}"]), (name, dep)


@pytest.mark.parametrize("name", G.kats())
def test_kernel_select_and_classify(name):
    k = G.kat(name)
    v = k["v"]
    sample = torch.from_numpy(k["sample"].view(np.int64)).cuda()
    tree, inorder, tpos, eqb = D.select_splitters(sample, v)
    assert np.array_equal(tree.cpu().numpy().view(np.uint64)[1:], k["tree"][1:])
    assert np.array_equal(inorder.cpu().numpy().view(np.uint64), k["inorder"])
    assert np.array_equal(tpos.cpu().numpy(), k["term_pos"])
    want_eqb = 2 * k["eq_leftmost"][k["node_to_inorder"][1:]] + 1
    assert np.array_equal(eqb.cpu().numpy()[1:].astype(np.int64), want_eqb)
    keys = torch.from_numpy(k["keys"].view(np.int64)).cuda()
    for variant in ("unroll", "equal"):
        got = D.classify(keys, tree, eqb, v, variant).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, k["oracle"]), variant


def _clusters(n, seed=1, prefix_len=8, clusters=4):
    rng = np.random.default_rng(seed)
    pre = [bytes(rng.integers(97, 123, size=prefix_len, dtype=np.uint8)) for _ in range(clusters)]
    return P.from_strings(
        pre[int(rng.integers(0, clusters))]
        + bytes(rng.integers(33, 127, size=int(rng.integers(1, 8)), dtype=np.uint8))
        for _ in range(n))


def test_step_hook_equality_buckets_advance_by_word():
    # test_ssss.py:205-217 restated
    s = _clusters(4000)
    records = []
    res = P.s5_sort(s, want_lcps=True, t_medium=512, step_hook=records.append)
    h, lcps, _ = oracle.s5_sort(s.buffer, s.handles)
    assert np.array_equal(res.set.handles, h) and np.array_equal(res.lcps, lcps)
    assert records
    root = records[0]
    assert (root.child_depths[1::2] == root.depth + 8).all()
    assert [r for r in records[1:] if r.depth == 8]


def test_step_hook_bucket_lcp_property():
    # Eq. 1 (test_ssss.py:231-256 restated): members of every bucket share
    # at least the documented prefix credit
    buf, hnd = corpora.gen_random(10_000, 13)
    s = P.StringSet(buf.tobytes(), hnd)
    records = []
    res = P.s5_sort(s, t_medium=1024, step_hook=records.append)
    rng = np.random.default_rng(0)
    checked = 0
    for rec in records:
        for i in range(rec.tree.num_buckets):
            lo, hi = rec.lo + int(rec.bounds[i]), rec.lo + int(rec.bounds[i + 1])
            if hi - lo < 2:
                continue
            credit = int(rec.child_depths[i])
            for a, b in rng.integers(lo, hi, size=(min(20, hi - lo), 2)):
                assert oracle.lcp(s.buffer, res.handles[a], res.handles[b]) >= credit
                checked += 1
    assert checked > 100


def test_step_hook_full_tree_root():
    # a root with the full v = 8191 tree (the cluster-sampled root step and the
    # root classify that builds the work records) seen through the hook:
    # bounds cover the input, Eq. 1 credits hold, output equals the oracle
    # (GPU-sized trees reach v = 8191 above 8192 x SEG_TARGET strings)
    buf, hnd = corpora.gen_random(9_000_000, 21)
    s = P.StringSet(buf.tobytes(), hnd)
    records = []
    res = P.s5_sort(s, want_lcps=True, step_hook=records.append)
    h, lcps, _ = oracle.parallel_s5(s.buffer, s.handles)
    assert np.array_equal(res.set.handles, h) and np.array_equal(res.lcps, lcps)
    root = records[0]
    assert root.lo == 0 and root.hi == len(hnd) and root.tree.num_buckets == 2 * 8191 + 1
    assert root.bounds[0] == 0 and root.bounds[-1] == len(hnd)
    assert (np.diff(root.bounds) >= 0).all()
    rng = np.random.default_rng(1)
    for i in rng.integers(0, root.tree.num_buckets, size=400):
        lo, hi = int(root.bounds[i]), int(root.bounds[i + 1])
        if hi - lo >= 2:
            assert oracle.lcp(s.buffer, res.set.handles[lo], res.set.handles[hi - 1]) >= int(root.child_depths[i])


def _oracle_tree(rec_tree):
    """The step record's splitter tree as the oracle's Tree (same fields)."""
    t = rec_tree
    return oracle.Tree(t.v, np.ascontiguousarray(t.tree, dtype=np.uint64),
                       np.ascontiguousarray(t.inorder, dtype=np.uint64),
                       np.ascontiguousarray(t.node_to_inorder, dtype=np.int64),
                       np.ascontiguousarray(t.slcp, dtype=np.int64),
                       np.asarray(t.eq_final, dtype=bool),
                       np.ascontiguousarray(t.eq_leftmost, dtype=np.int64),
                       np.ascontiguousarray(t.term_pos, dtype=np.int64))


@pytest.mark.parametrize("variant", ["unroll", "equal"])
@pytest.mark.parametrize("gen,n,t_medium", [("clusters", 6000, 512), ("random", 300_000, 2048),
                                            ("urls", 60_000, 1024)])
def test_step_bounds_match_oracle_classify_distribute(gen, n, t_medium, variant):
    """Per-step parity: every step's bucket bounds equal
    those the oracle's classify_keys + distribute (ssss.py:149-212) produce
    for the same strings at the same depth with the SAME splitters, and the
    step's stable scatter leaves every bucket's strings in the order
    distribute gives them wherever the step's output is still visible
    (buckets that are final after the step)."""
    if gen == "clusters":
        s = _clusters(n)
    elif gen == "random":
        buf, hnd = corpora.gen_random(n, 5)
        s = P.StringSet(buf.tobytes(), hnd)
    else:
        buf, hnd = corpora.gen_urls(n)
        s = P.StringSet(buf.tobytes(), hnd)
    records = []
    res = P.s5_sort(s, want_lcps=True, t_medium=t_medium, variant=variant,
                    step_hook=records.append)
    out_h = res.set.handles
    assert records
    buf_np = np.frombuffer(s.buffer, dtype=np.uint8) if isinstance(s.buffer, (bytes, bytearray)) \
        else np.asarray(s.buffer)
    for rec in records:
        # the segment's strings are exactly the final output's [lo, hi)
        seg = np.ascontiguousarray(out_h[rec.lo:rec.hi], dtype=np.int64)
        keys = oracle.extract_keys(buf_np, seg, rec.depth)
        tree = _oracle_tree(rec.tree)
        ids = oracle.classify_keys(keys, tree, variant)
        _, bounds = oracle.distribute(seg, ids, tree.num_buckets)
        assert np.array_equal(np.asarray(rec.bounds, dtype=np.int64), bounds), \
            f"step [{rec.lo},{rec.hi}) depth {rec.depth}: bucket bounds differ from the oracle"
        # the final order is bucket-major: ids of the sorted segment are non-decreasing
        assert (np.diff(ids) >= 0).all()


def test_hook_errors_propagate():
    s = _clusters(3000)

    def boom(rec):
        raise KeyError("hook exploded")

    with pytest.raises(KeyError, match="hook exploded"):
        P.s5_sort(s, t_medium=64, step_hook=boom)


def test_sort_host_abi_matches_device_path():
    buf, hnd = corpora.gen_urls(20_000, hosts=200, pool=8)
    oh, ol, od = D.sort_host(buf, hnd, want_lcps=True, want_dchar=True)
    h, lcps, _ = oracle.parallel_s5(buf, hnd)
    assert np.array_equal(oh, h) and np.array_equal(ol, lcps)
    assert np.array_equal(od, oracle.fill_dchar(buf, h, lcps))


SCALED = [("c1_random", 1.0), ("c2_dna", 1 / 16), ("c3_urls", 1 / 16), ("c4_suffixes", 1 / 64),
          ("c5_nodup", 1 / 256)]


@pytest.mark.parametrize("cfg,scale", SCALED)
def test_config_parity_scaled(cfg, scale):
    buf, hnd = corpora.CONFIGS[cfg](scale)
    ds = D.upload(buf, hnd)
    out_h, lcps, _ = D.sort(ds, want_lcps=True)
    h, l, _ = oracle.parallel_s5(buf, hnd)
    got_h = out_h.cpu().numpy()
    assert np.array_equal(got_h, h)
    assert np.array_equal(lcps.cpu().numpy(), l)


@pytest.mark.parametrize("n", [32769, 40000, 8192 * 148 * 2 + 7, 9_000_000])
@pytest.mark.parametrize("alphabet", [2, 4, 26])
def test_root_step_sizes_vs_oracle(n, alphabet):
    """Roots just above the fused-CTA limit (device-wide root with few tiles),
    around the small-root tile spreading limit (2 x SMs x MIN_TILE), and
    above 8192 x SEG_TARGET (the full v = 8191 tree drawn by the cluster
    root sample); small alphabets make most scatter rounds collide inside a
    32-string round."""
    rng = np.random.default_rng(n + alphabet)
    lens = rng.integers(0, 14, size=n).astype(np.int64)
    off = np.zeros(n, dtype=np.int64)
    np.cumsum(lens[:-1] + 1, out=off[1:])
    buf = np.zeros(int(lens.sum()) + n, dtype=np.uint8)
    chars = (97 + rng.integers(0, alphabet, size=int(lens.sum()))).astype(np.uint8)
    mask = np.ones(len(buf), dtype=bool)
    mask[off + lens] = False
    buf[mask] = chars
    hnd = rng.permutation(off) if alphabet == 4 else off
    ds = D.upload(buf, hnd)
    h, l, _ = D.sort(ds, want_lcps=True)
    oh, ol, _ = oracle.parallel_s5(buf, hnd)
    assert np.array_equal(h.cpu().numpy(), oh)
    assert np.array_equal(l.cpu().numpy(), ol)


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0] * 8])
@pytest.mark.parametrize("name", ["random_3000", "dups_2000", "shuffled_dups_2500", "urls_2000",
                                  "all_equal_700", "suffixes_1800", "random_n2", "random_n17"])
def test_parallel_s5_multi_device_partition(name, devices):
    """parallel_s5 with p parts (s5g_sort_multi): sample-sort partition by
    string splitters with input-position ties, one sort per part, boundary
    LCPs fixed on the host.  One GPU here, so the parts share device 0 -- the
    partition, the per-part offsets and the boundary fix-up are what is
    tested; the output must equal the reference's bit for bit."""
    c = G.case(name)
    s = P.StringSet(c["buffer_bytes"], c["handles"])
    res = P.parallel_s5(s, want_lcps=True, want_dchar=True, devices=devices)
    assert np.array_equal(res.set.handles, c["out_handles"])
    assert np.array_equal(res.lcps, c["lcps"])
    assert np.array_equal(res.dchar, c["dchar"])
    out = P.parallel_s5(s, devices=devices)
    assert np.array_equal(out.handles, c["out_handles"])


def test_parallel_s5_multi_device_scaled_config():
    buf, hnd = corpora.gen_urls(1 << 18, 7)
    s = P.StringSet(buf.tobytes(), hnd)
    res = P.parallel_s5(s, want_lcps=True, devices=[0, 0, 0, 0])
    h, l, _ = oracle.parallel_s5(buf, hnd)
    assert np.array_equal(res.set.handles, h) and np.array_equal(res.lcps, l)


def test_parallel_s5_p_counts_gpus():
    c = G.case("random_3000")
    s = P.StringSet(c["buffer_bytes"], c["handles"])
    ndev = torch.cuda.device_count()
    res = P.parallel_s5(s, p=None, want_lcps=True)  # p=None: every visible GPU
    assert np.array_equal(res.set.handles, c["out_handles"])
    with pytest.raises(ValueError, match="exceeds"):
        P.parallel_s5(s, p=ndev + 1)
    with pytest.raises(ValueError, match="at least 1"):
        P.parallel_s5(s, p=0)


def test_host_entry_rejects_handles_outside_the_buffer():
    """The reference's input errors through the host entry (s5g_sort_host
    checks handle bounds on the device): ValueError, no crash."""
    s = P.StringSet(b"ab\0cd\0", np.array([0, 3, 6], dtype=np.int64))
    with pytest.raises(ValueError, match="outside the buffer"):
        P.s5_sort(s, want_lcps=True)
    s = P.StringSet(b"ab\0cd\0", np.array([0, -1], dtype=np.int64))
    with pytest.raises(ValueError, match="outside the buffer"):
        P.s5_sort(s)
    s = P.StringSet(b"ab\0cd", np.array([0, 3], dtype=np.int64))
    with pytest.raises(ValueError, match="not zero-terminated"):
        P.s5_sort(s)
