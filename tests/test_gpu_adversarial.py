"""Adversarial shapes on the GPU path, checked by the oracle's K11 certificate
(permutation, order, stability of ties, exact LCPs): long identical
strings (device-level equality chains), long shared prefixes with short
distinguishing tails, one very long string, all byte values, heavy
duplication at scale."""

import time

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_1403_2056_b200 import device as D  # noqa: E402


def _pack(lens, fill):
    n = len(lens)
    off = np.zeros(n, dtype=np.int64)
    if n:
        np.cumsum(lens[:-1] + 1, out=off[1:])
    buf = np.zeros(int(lens.sum()) + n, dtype=np.uint8)
    for i in range(n):
        buf[off[i]:off[i] + lens[i]] = fill(i, int(lens[i]))
    return buf, off


def _check(buf, hnd, limit_s=None):
    ds = D.upload(buf, hnd)
    t0 = time.time()
    h, l, _ = D.sort(ds, want_lcps=True)
    torch.cuda.synchronize()
    dt = time.time() - t0
    st, bad = oracle.certify(buf, hnd, h.cpu().numpy(), l.cpu().numpy())
    assert st == 0, (oracle.CERT_STATUS[st], bad)
    if limit_s is not None:
        assert dt < limit_s, dt
    return dt


def test_identical_long_strings():
    n, L = 1 << 18, 300
    s = np.frombuffer(b"ab" * 150, dtype=np.uint8)
    buf = np.tile(np.r_[s, 0].astype(np.uint8), n)
    hnd = np.arange(n, dtype=np.int64) * (L + 1)
    _check(buf, hnd)


def test_long_shared_prefix_short_tails():
    rng = np.random.default_rng(1)
    n, P = 1 << 16, 2000
    prefix = rng.integers(97, 123, size=P, dtype=np.uint8)
    tails = rng.integers(97, 100, size=(n, 6), dtype=np.uint8)
    buf = np.zeros((n, P + 7), dtype=np.uint8)
    buf[:, :P] = prefix
    buf[:, P:P + 6] = tails
    _check(buf.reshape(-1), np.arange(n, dtype=np.int64) * (P + 7))


def test_one_very_long_string_among_short():
    rng = np.random.default_rng(2)
    lens = rng.integers(0, 12, size=50_000).astype(np.int64)
    lens[777] = 1 << 20
    lens[778] = (1 << 20) - 1
    big = rng.integers(97, 99, size=1 << 20, dtype=np.uint8)
    buf, off = _pack(lens, lambda i, L: big[:L] if L > 100 else rng.integers(97, 99, size=L, dtype=np.uint8))
    _check(buf, off)


def test_all_byte_values_and_lengths():
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 300, size=200_000).astype(np.int64)
    total = int(lens.sum())
    chars = rng.integers(1, 256, size=total, dtype=np.uint8)
    pos = np.r_[0, np.cumsum(lens)]
    buf, off = _pack(lens, lambda i, L: chars[pos[i]:pos[i] + L])
    _check(buf, off)


def test_heavy_duplication_shuffled_handles():
    rng = np.random.default_rng(4)
    words = [bytes(rng.integers(97, 123, size=int(rng.integers(1, 40)), dtype=np.uint8)) for _ in range(300)]
    items = [words[int(k)] for k in rng.integers(0, 300, size=1 << 21)]
    buf = np.frombuffer(b"".join(w + b"\0" for w in items), dtype=np.uint8)
    off = np.r_[0, np.cumsum([len(w) + 1 for w in items])[:-1]].astype(np.int64)
    _check(buf, rng.permutation(off))


def test_full_width_tiles_with_one_bucket():
    """A full-width (16 383-bucket) root over enough strings for the widest
    classify / scatter tiles (WIDE_TILE = 65 280 strings, n >= 4 x 148 tiles)
    whose strings nearly all fall into ONE equality bucket: every tile's
    count of that bucket is the tile size, the largest value the packed u16
    per-tile counts must hold."""
    n = 65280 * 4 * 148 + 12345
    rng = np.random.default_rng(7)
    buf = np.zeros((n, 4), dtype=np.uint8)
    buf[:, :3] = np.frombuffer(b"abc", dtype=np.uint8)
    odd = rng.integers(0, n, size=5000)
    buf[odd, :3] = rng.integers(97, 123, size=(5000, 3), dtype=np.uint8)
    _check(buf.reshape(-1), np.arange(n, dtype=np.int64) * 4)


@pytest.mark.parametrize("n", [3000, 20000, 30000, 200000])
def test_keys_equal_to_the_tree_padding(n):
    """Words of eight 0xFF bytes equal the ~0 padding that fills a fused
    step's splitter tree above its real splitters (med_plan): they must land
    in one all-equal bucket a word deeper, next to smaller and terminated
    keys, at fused-step sizes (the first step of an input <= 32768 strings is
    a fused one) and below a device-wide root."""
    rng = np.random.default_rng(n)
    kinds = rng.integers(0, 4, size=n)
    strs = []
    for k in kinds:
        tail = bytes(rng.integers(250, 256, size=int(rng.integers(0, 12)), dtype=np.uint8))
        if k == 0:
            strs.append(b"\xff" * 8 + tail)              # word 0 == ~0
        elif k == 1:
            strs.append(b"\xff" * 16 + tail)             # words 0 and 1 == ~0
        elif k == 2:
            strs.append(b"\xff" * int(rng.integers(0, 8)))  # terminated inside word 0
        else:
            strs.append(bytes(rng.integers(1, 256, size=8, dtype=np.uint8)) + tail)
    buf = np.frombuffer(b"".join(s + b"\0" for s in strs), dtype=np.uint8).copy()
    hnd = np.concatenate(([0], np.cumsum([len(s) + 1 for s in strs])[:-1])).astype(np.int64)
    _check(buf, hnd)
