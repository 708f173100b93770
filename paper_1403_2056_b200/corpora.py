"""Seeded synthetic corpora for the five BASELINE.json configurations.

The paper's data sets (URL crawl, GOV2, Wikipedia, Sinha's DNA / NoDup) are
not available; these frozen generators stand in for them with the shapes,
sizes and value distributions BASELINE.json names:

  C1  random   : exactly strsort.bench.gen_random(n, seed) (bench.py:31-46):
                 lengths U[0,20), bytes U[33,127)
  C2  dna      : n = 2^24 reads of length 100 over ACGT with p = .3/.2/.2/.3
  C3  urls     : n = 2^23 'http://' + Zipf(1.1) host from 10,000 seeded hosts
                 + 1-4 '/'-segments from a finite per-host pool (duplicates)
  C4  suffixes : all 2^24 suffixes of an order-2 Markov text over a-z with
                 5% of the text overwritten by copies of earlier 1-4 KB blocks
  C5  nodup    : n = 2^28, lengths U[32,200]: 16-char prefix from a 2^16-word
                 vocabulary + lowercase filler + unique 6-char base-36 counter;
                 counter-based (csrc/s5g_gen.cu), host and device generators

Every generator returns (buffer: np.ndarray[uint8], handles: np.ndarray[int64]).
"""

from __future__ import annotations

import numpy as np

ALPHA = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", dtype=np.uint8)
B36 = np.frombuffer(b"0123456789abcdefghijklmnopqrstuvwxyz", dtype=np.uint8)


def _pack_lengths(lens: np.ndarray, fill) -> tuple[np.ndarray, np.ndarray]:
    """Buffer of zero-terminated strings with the given lengths; fill(total)
    returns the characters in order."""
    n = len(lens)
    total = int(lens.sum())
    offsets = np.zeros(n, dtype=np.int64)
    if n:
        np.cumsum(lens[:-1] + 1, out=offsets[1:])
    buf = np.zeros(total + n, dtype=np.uint8)
    chars = fill(total)
    mask = np.ones(total + n, dtype=bool)
    mask[offsets + lens] = False
    buf[mask] = chars
    return buf, offsets


def gen_random(n: int = 1_000_000, seed: int = 0):
    """C1: identical bytes to strsort.bench.gen_random(n, seed)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 20, size=n, dtype=np.int64)
    total = int(lens.sum())
    chars = rng.integers(33, 127, size=total, dtype=np.uint8).astype(np.uint8)
    return _pack_lengths(lens, lambda t: chars)


def gen_dna(n: int = 1 << 24, length: int = 100, seed: int = 1):
    """C2: fixed-length reads, i.i.d. A/C/G/T with probabilities .3/.2/.2/.3."""
    rng = np.random.default_rng(seed)
    table = np.frombuffer(b"AAACCGGTTT", dtype=np.uint8)
    buf = np.zeros((n, length + 1), dtype=np.uint8)
    step = max(1, (1 << 26) // (length + 1))
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        buf[lo:hi, :length] = table[rng.integers(0, 10, size=(hi - lo, length), dtype=np.uint8)]
    return buf.reshape(-1), np.arange(n, dtype=np.int64) * (length + 1)


def _expand(pieces: np.ndarray, piece_off: np.ndarray, piece_len: np.ndarray,
            seq: np.ndarray, per_string: np.ndarray):
    """Concatenate piece ids `seq` (grouped per string by `per_string`
    counts) into a zero-terminated buffer."""
    plen = piece_len[seq]
    slen = np.add.reduceat(plen, np.r_[0, np.cumsum(per_string)[:-1]]) if len(seq) else plen
    n = len(per_string)
    str_off = np.zeros(n, dtype=np.int64)
    np.cumsum(slen[:-1] + 1, out=str_off[1:])
    # output offset of every piece occurrence
    first_piece = np.r_[0, np.cumsum(per_string)[:-1]]
    within = np.arange(len(seq), dtype=np.int64) - np.repeat(first_piece, per_string)
    pcum = np.cumsum(plen) - plen  # global exclusive prefix of piece lengths
    str_piece_base = pcum[first_piece]
    piece_out = np.repeat(str_off, per_string) + (pcum - np.repeat(str_piece_base, per_string))
    del within
    total = int(str_off[-1] + slen[-1] + 1)
    buf = np.zeros(total, dtype=np.uint8)
    # byte-level gather, in chunks to bound memory
    CH = 1 << 22
    for lo in range(0, len(seq), CH):
        hi = min(len(seq), lo + CH)
        pl = plen[lo:hi]
        src = np.repeat(piece_off[seq[lo:hi]], pl)
        dst = np.repeat(piece_out[lo:hi], pl)
        k = np.arange(len(src), dtype=np.int64) - np.repeat(np.cumsum(pl) - pl, pl)
        buf[dst + k] = pieces[src + k]
    return buf, str_off


def gen_urls(n: int = 1 << 23, seed: int = 2, hosts: int = 10_000, pool: int = 16_000,
             zipf_s: float = 1.1):
    """C3: URL-like strings: 'http://' + a Zipf(zipf_s)-popular host (from
    `hosts` seeded names of 8-20 letters + '.com') + 1-4 '/'-segments of 3-12
    letters drawn from one seeded pool of `pool` segments shared by all hosts.
    The finite pool makes popular hosts repeat short URLs: at n = 2^23 the
    frozen parameters give ~10% duplicates and a mean LCP of ~30 (BASELINE
    configs[2]; the achieved figures are in DESIGN.md §5)."""
    rng = np.random.default_rng(seed)
    # piece table: [0] 'http://', hosts, then the '/'+segment pool
    texts: list[bytes] = [b"http://"]
    hlen = rng.integers(8, 21, size=hosts)
    for L in hlen:
        texts.append(bytes(ALPHA[rng.integers(0, 26, size=int(L))]) + b".com")
    seg_base = len(texts)
    slen = rng.integers(3, 13, size=pool)
    for L in slen:
        texts.append(b"/" + bytes(ALPHA[rng.integers(0, 26, size=int(L))]))
    piece_len = np.array([len(t) for t in texts], dtype=np.int64)
    piece_off = np.r_[0, np.cumsum(piece_len)[:-1]].astype(np.int64)
    pieces = np.frombuffer(b"".join(texts), dtype=np.uint8)
    ranks = np.arange(1, hosts + 1, dtype=np.float64)
    p = ranks ** -zipf_s
    p /= p.sum()
    host = rng.choice(hosts, size=n, p=p)
    nseg = rng.integers(1, 5, size=n)
    per = 2 + nseg
    seq = np.empty(int(per.sum()), dtype=np.int64)
    start = np.r_[0, np.cumsum(per)[:-1]]
    seq[start] = 0
    seq[start + 1] = 1 + host
    for j in range(4):
        has = nseg > j
        seq[start[has] + 2 + j] = seg_base + rng.integers(0, pool, size=int(has.sum()))
    return _expand(pieces, piece_off, piece_len, seq, per)


def gen_suffix_markov(n: int = 1 << 24, seed: int = 3, copy_frac: float = 0.05,
                      chains: int = 1024):
    """C4: suffixes of an order-2 Markov text with copied 1-4 KB blocks.

    The text is generated as `chains` independent order-2 chains (seeded
    transition table, Dirichlet(0.3) rows) laid end to end, then 5% of it is
    overwritten, left to right, by copies of earlier 1024-4096-byte blocks."""
    rng = np.random.default_rng(seed)
    trans = rng.dirichlet(np.full(26, 0.3), size=26 * 26)
    cdf = np.cumsum(trans, axis=1)
    cdf[:, -1] = 1.0
    per = (n + chains - 1) // chains
    text = np.zeros((chains, per), dtype=np.uint8)
    a = rng.integers(0, 26, size=chains)
    b = rng.integers(0, 26, size=chains)
    u = rng.random(size=(per, chains))
    for t in range(per):
        row = cdf[a * 26 + b]
        c = (row < u[t][:, None]).sum(axis=1)
        c = np.minimum(c, 25)
        text[:, t] = c
        a, b = b, c
    text = text.reshape(-1)[:n]
    copied = 0
    target = int(copy_frac * n)
    hi_len = max(2, min(4097, n // 4))
    while copied < target:
        L = int(rng.integers(min(1024, hi_len - 1), hi_len))
        p = int(rng.integers(L + 1, n - L))
        q = int(rng.integers(0, p - L))
        text[p:p + L] = text[q:q + L]
        copied += L
    buf = np.empty(n + 1, dtype=np.uint8)
    buf[:n] = ALPHA[text]
    buf[n] = 0
    return buf, np.arange(n, dtype=np.int64)


_gen_lib = None


def _gen():
    """libs5gen.so (csrc/s5g_gen.cu): the counter-based C5 generator."""
    global _gen_lib
    if _gen_lib is None:
        import ctypes as C

        from .build import GEN_PATH

        if not GEN_PATH.exists():
            raise ImportError(f"{GEN_PATH} is missing: build it with "
                              "`python -m paper_1403_2056_b200.build`")
        L = C.CDLL(str(GEN_PATH))
        i64, u64, p = C.c_int64, C.c_uint64, C.c_void_p
        L.s5gen_nodup_bytes.restype = i64
        L.s5gen_nodup_bytes.argtypes = [i64, i64, u64]
        L.s5gen_nodup_host.restype = C.c_int
        L.s5gen_nodup_host.argtypes = [i64, i64, u64, p, p]
        L.s5gen_nodup_device.restype = C.c_int
        L.s5gen_nodup_device.argtypes = [i64, i64, u64, p, p, p]
        L.s5gen_last_error.restype = C.c_char_p
        _gen_lib = L
    return _gen_lib


def _gen_check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("s5gen: " + _gen().s5gen_last_error().decode())


def nodup_bytes(n: int, seed: int = 4) -> int:
    """Arena length (terminators included) of the first n C5 strings."""
    return int(_gen().s5gen_nodup_bytes(0, n, seed))


def gen_nodup(n: int = 1 << 28, seed: int = 4, out: np.ndarray | None = None):
    """C5: unique strings, lengths U[32,200]: 16-char prefix from a 2^16-word
    vocabulary, lowercase filler, 6-char base-36 counter (36^6 > 2^28 keeps
    them unique).  Counter-based (csrc/s5g_gen.cu): every byte is a function
    of (seed, string index, position), so gen_nodup(m) is a prefix of
    gen_nodup(n) for m <= n and gen_nodup_device writes the same bytes.
    Generated on all host cores (OpenMP); `out` (uint8, >= nodup_bytes(n))
    may be a pinned buffer."""
    total = nodup_bytes(n, seed)
    buf = out[:total] if out is not None else np.empty(total, dtype=np.uint8)
    assert buf.dtype == np.uint8 and buf.size == total and buf.flags.c_contiguous
    hnd = np.empty(n, dtype=np.int64)
    _gen_check(_gen().s5gen_nodup_host(0, n, seed, buf.ctypes.data if total else None,
                                       hnd.ctypes.data if n else None))
    return buf, hnd


def gen_nodup_device(n: int = 1 << 28, seed: int = 4, device=None, n0: int = 0):
    """C5 generated directly in HBM (same bytes as gen_nodup): strings
    n0 .. n0+n-1 (a rank's contiguous slice of the corpus when n0 > 0), as
    (arena uint8 tensor padded with zeros past arena_len, arena_len, handles
    int64 tensor relative to the slice) -- the device.DeviceStrings fields."""
    import torch

    from ._lib import S5G_ARENA_PAD

    dev = device or torch.device("cuda", torch.cuda.current_device())
    total = int(_gen().s5gen_nodup_bytes(n0, n, seed))
    cap = (total + S5G_ARENA_PAD + 15) // 16 * 16
    arena = torch.empty(cap, dtype=torch.uint8, device=dev)
    arena[total:].zero_()
    hnd = torch.empty(max(n, 1), dtype=torch.int64, device=dev)[:n]
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        _gen_check(_gen().s5gen_nodup_device(n0, n, seed, arena.data_ptr(), hnd.data_ptr(), st))
    return arena, total, hnd


CONFIGS = {
    "c1_random": lambda scale=1.0: gen_random(int(1_000_000 * scale), 0),
    "c2_dna": lambda scale=1.0: gen_dna(int((1 << 24) * scale), 100, 1),
    "c3_urls": lambda scale=1.0: gen_urls(int((1 << 23) * scale), 2),
    "c4_suffixes": lambda scale=1.0: gen_suffix_markov(int((1 << 24) * scale), 3),
    "c5_nodup": lambda scale=1.0: gen_nodup(int((1 << 28) * scale), 4),
}
