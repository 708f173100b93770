"""Generate the golden vectors that pin the oracle and the GPU path.

Runs the REFERENCE implementation (strsort 0.1.0, imported from
/root/reference/pkg/src -- only available in the build container) on small
seeded corpora and records inputs and outputs into ``golden_s5.npz``.  The
corpora builders below are this repo's own; they reproduce the *shapes* the
reference tests use (random, all-equal, all-empty, shared 8-char prefix
clusters, suffixes, URL-like, deep shared prefixes, heavy duplicates,
shuffled handles, high bytes, depth > 0).

Usage:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden_s5.npz"


def pack(items: list[bytes]) -> tuple[bytes, np.ndarray]:
    offs, pos = [], 0
    for s in items:
        offs.append(pos)
        pos += len(s) + 1
    return b"".join(s + b"\0" for s in items), np.asarray(offs, dtype=np.int64)


def corpora() -> dict[str, tuple[bytes, np.ndarray, int]]:
    """name -> (buffer, handles, depth)"""
    out = {}
    rng = np.random.default_rng(2024)

    def rand_items(n, max_len, lo, hi):
        return [bytes(rng.integers(lo, hi, size=int(rng.integers(0, max_len)), dtype=np.uint8))
                for _ in range(n)]

    for n in (0, 1, 2, 3, 17, 64, 65):
        out[f"random_n{n}"] = (*pack(rand_items(n, 20, 33, 127)), 0)
    out["random_3000"] = (*pack(rand_items(3000, 20, 33, 127)), 0)
    out["random_long_2000"] = (*pack(rand_items(2000, 60, 97, 100)), 0)
    out["all_equal_700"] = (*pack([b"abcdefghijxyz"] * 700), 0)
    out["all_equal_8_300"] = (*pack([b"abcdefgh"] * 300), 0)
    out["all_empty_300"] = (*pack([b""] * 300), 0)
    pre = [bytes(rng.integers(97, 123, size=8, dtype=np.uint8)) for _ in range(4)]
    items = [pre[int(rng.integers(0, 4))] +
             bytes(rng.integers(33, 127, size=int(rng.integers(1, 8)), dtype=np.uint8))
             for _ in range(2500)]
    out["clusters_2500"] = (*pack(items), 0)
    text = bytes(rng.integers(97, 101, size=1800, dtype=np.uint8))
    out["suffixes_1800"] = (text + b"\0", np.arange(1800, dtype=np.int64), 0)
    hosts = [b"www.alpha.com", b"www.alpha.org", b"db.beta.net", b"gamma.io"]
    segs = [b"news", b"img/static", b"a/b", b"idx"]
    items = [b"http://" + hosts[int(rng.integers(0, 4))] + b"/" + segs[int(rng.integers(0, 4))]
             + b"/p" + str(int(rng.integers(0, 300))).encode() for _ in range(2000)]
    out["urls_2000"] = (*pack(items), 0)
    base = bytes(rng.integers(97, 123, size=70, dtype=np.uint8))
    items = [base[: int(rng.integers(30, 70))] +
             bytes(rng.integers(97, 99, size=int(rng.integers(0, 12)), dtype=np.uint8))
             for _ in range(1500)]
    out["deep_prefix_1500"] = (*pack(items), 0)
    out["dups_2000"] = (*pack(rand_items(2000, 5, 97, 99)), 0)
    buf, h = pack(rand_items(2500, 12, 97, 101))
    out["shuffled_dups_2500"] = (buf, rng.permutation(h), 0)
    out["high_bytes_1500"] = (*pack(rand_items(1500, 14, 1, 256)), 0)
    items = [b"pre" + s for s in rand_items(900, 10, 97, 102)]
    out["depth3_900"] = (*pack(items), 3)
    # copies of long blocks inside a suffix text: LCPs well beyond 8 words
    t = bytearray(rng.integers(97, 100, size=3000, dtype=np.uint8).tobytes())
    t[2000:2400] = t[100:500]
    out["suffix_copies_3000"] = (bytes(t) + b"\0", np.arange(3000, dtype=np.int64), 0)
    return out


def main() -> None:
    sys.path.insert(0, str(REF))
    from strsort import ssss, strset, mkqs, basecase  # noqa: E402
    from strsort.parallel import parallel_s5  # noqa: E402

    arrays: dict[str, np.ndarray] = {}
    meta = {"reference": "strsort 0.1.0 (/root/reference/pkg)", "cases": {}}
    for name, (buf, handles, depth) in corpora().items():
        sset = strset.StringSet(buf, handles)
        res = ssss.s5_sort(sset, depth=depth, want_lcps=True, want_dchar=True)
        for kw in ({"t_medium": 16}, {"t_medium": 256, "variant": "equal"}, {"seed": 9}):
            alt = ssss.s5_sort(sset, depth=depth, want_lcps=True, **kw)
            assert np.array_equal(alt.set.handles, res.set.handles), (name, kw)
            assert np.array_equal(alt.lcps, res.lcps), (name, kw)
        if depth == 0 and len(handles) >= 2:
            par = parallel_s5(sset, p=2, want_lcps=True, t_medium=256)
            assert np.array_equal(par.set.handles, res.set.handles), name
            assert np.array_equal(par.lcps, res.lcps), name
            # the reference output is the stable content sort
            stable = sorted(range(len(handles)), key=lambda i: sset.string_at(i))
            assert np.array_equal(handles[stable], res.set.handles), name
        arrays[f"{name}/buffer"] = np.frombuffer(buf, dtype=np.uint8)
        arrays[f"{name}/handles"] = handles
        arrays[f"{name}/out_handles"] = res.set.handles
        arrays[f"{name}/lcps"] = res.lcps
        arrays[f"{name}/dchar"] = res.dchar
        case = {"n": int(len(handles)), "depth": depth}
        if depth == 0:
            mk = mkqs.mkqs_cached(sset)
            assert np.array_equal(mk.lcps, res.lcps)
            arrays[f"{name}/mkqs_handles"] = mk.set.handles
            case["mkqs_word_fetches"] = mk.stats.word_fetches
            if len(handles) <= 300:
                ins = basecase.lcp_insertion_sort(sset)
                arrays[f"{name}/ins_handles"] = ins.set.handles
                arrays[f"{name}/ins_lcps"] = ins.lcps
                case["ins_char_cmps"] = ins.stats.char_cmps
            d = strset.dist_stats(sset)
            case["D"], case["L"] = d.D, d.L
            for dep in (0, 2, 5, 9):
                arrays[f"{name}/keys_d{dep}"] = strset.extract_keys(sset, handles, dep)
        meta["cases"][name] = case

    # K-way LCP merge (lcpmerge.py) and partitioned_merge_sort (parallel.py:885)
    from strsort import lcpmerge  # noqa: E402
    from strsort.parallel import partitioned_merge_sort  # noqa: E402
    merge_cases = {}
    for name in ("random_n17", "random_3000", "urls_2000", "dups_2000", "deep_prefix_1500",
                 "suffixes_1800", "all_equal_700", "shuffled_dups_2500", "high_bytes_1500"):
        buf = arrays[f"{name}/buffer"].tobytes()
        handles = arrays[f"{name}/handles"]
        sset = strset.StringSet(buf, handles)
        for K in (2, 3, 5):
            cuts = np.linspace(0, len(handles), K + 1).astype(np.int64)
            streams, hs, ls, cs = [], [], [], []
            for j in range(K):
                sub = sset.with_handles(handles[cuts[j]:cuts[j + 1]])
                r = ssss.s5_sort(sub, want_lcps=True, want_dchar=True)
                streams.append(lcpmerge.LcpStream(sset, r.set.handles, r.lcps, r.dchar))
                hs.append(r.set.handles), ls.append(r.lcps), cs.append(r.dchar)
            h0, l0 = lcpmerge.kway_lcp_merge(streams, cached=False)
            h1, l1 = lcpmerge.kway_lcp_merge(streams, cached=True)
            assert np.array_equal(h0, h1) and np.array_equal(l0, l1), (name, K)
            assert np.array_equal(h0, arrays[f"{name}/out_handles"]), (name, K)
            assert np.array_equal(l0, arrays[f"{name}/lcps"]), (name, K)
            pre = f"merge_{name}_k{K}"
            arrays[f"{pre}/run_off"] = cuts
            arrays[f"{pre}/run_handles"] = np.concatenate(hs)
            arrays[f"{pre}/run_lcps"] = np.concatenate(ls)
            arrays[f"{pre}/run_dchar"] = np.concatenate(cs)
            arrays[f"{pre}/out_handles"] = h0
            arrays[f"{pre}/out_lcps"] = l0
            merge_cases[pre] = {"case": name, "K": K}
        pm = partitioned_merge_sort(sset, K=4, p=2, want_lcps=True, t_medium=512)
        assert np.array_equal(pm.set.handles, arrays[f"{name}/out_handles"]), name
        assert np.array_equal(pm.lcps, arrays[f"{name}/lcps"]), name
    meta["merge"] = merge_cases

    # splitter-tree / classify / distribute known answers
    rng = np.random.default_rng(7)
    kat = {}
    for i, (v, count, alphabet) in enumerate([(3, 7, 256), (7, 15, 4), (15, 31, 3), (63, 127, 20),
                                              (255, 511, 2), (1023, 2047, 1000), (8191, 16383, 50),
                                              (8191, 16383, 1 << 40), (31, 63, 1)]):
        raw = rng.integers(1, alphabet + 1, size=count, dtype=np.uint64) * np.uint64(0x0101010101)
        sample = np.sort(raw.astype(np.uint64))
        tree = ssss.select_splitters(sample, v)
        keys = np.concatenate([sample, rng.integers(0, 1 << 62, size=500, dtype=np.uint64),
                               sample[::3] + np.uint64(1)]).astype(np.uint64)
        oracle = ssss.classify_keys(keys, tree, "unroll")
        assert np.array_equal(oracle, ssss.classify_keys(keys, tree, "equal"))
        pre = f"kat{i}"
        arrays[f"{pre}/sample"] = sample
        arrays[f"{pre}/keys"] = keys
        arrays[f"{pre}/oracle"] = oracle
        for fld in ("tree", "inorder", "node_to_inorder", "slcp", "eq_leftmost", "term_pos"):
            arrays[f"{pre}/{fld}"] = getattr(tree, fld)
        arrays[f"{pre}/eq_final"] = tree.eq_final.astype(np.uint8)
        hnd = np.arange(len(keys), dtype=np.int64) * 3
        out_h, bounds = ssss.distribute(hnd, oracle, tree.num_buckets)
        arrays[f"{pre}/dist_handles"] = out_h
        arrays[f"{pre}/dist_bounds"] = bounds
        kat[pre] = {"v": v}
    meta["kat"] = kat
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(meta['cases'])} cases)")


if __name__ == "__main__":
    main()
