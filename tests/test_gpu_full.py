"""Full-size parity on the BASELINE.json configurations.

C1-C3: bit-exact handles and LCPs against the pinned oracle (parallel S^5 on
all host cores).  C4 (2^24 suffixes, LCPs in the thousands) and C5 (scaled to
2^24 strings here): the K11 certificate -- permutation, order, stability of
ties and the exact LCP array, O(n + L) -- which defines the same unique
output.  Plus size-independent properties: idempotence (sorting the sorted
order is the identity) and invariance under shuffling the input."""

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")

from paper_1403_2056_b200 import corpora  # noqa: E402
from paper_1403_2056_b200 import device as D  # noqa: E402


def gpu_sort(buf, hnd, **kw):
    ds = D.upload(buf, hnd)
    h, l, _ = D.sort(ds, want_lcps=True, **kw)
    return h.cpu().numpy(), l.cpu().numpy()


@pytest.mark.parametrize("cfg", ["c1_random", "c2_dna", "c3_urls"])
def test_full_size_bit_exact(cfg):
    buf, hnd = corpora.CONFIGS[cfg](1.0)
    h, l = gpu_sort(buf, hnd)
    oh, ol, _ = oracle.parallel_s5(buf, hnd)
    assert np.array_equal(h, oh)
    assert np.array_equal(l, ol)


@pytest.mark.parametrize("cfg,scale", [("c4_suffixes", 1.0), ("c5_nodup", 1 / 16)])
def test_full_size_certificate(cfg, scale):
    buf, hnd = corpora.CONFIGS[cfg](scale)
    h, l = gpu_sort(buf, hnd)
    status, bad = oracle.certify(buf, hnd, h, l)
    assert status == 0, (oracle.CERT_STATUS[status], bad)


def test_idempotent_and_shuffle_invariant():
    buf, hnd = corpora.gen_urls(1 << 20, 5)
    h, l = gpu_sort(buf, hnd)
    h2, l2 = gpu_sort(buf, h)          # sorting the sorted order changes nothing
    assert np.array_equal(h2, h) and np.array_equal(l2, l)
    perm = np.random.default_rng(0).permutation(len(hnd))
    h3, l3 = gpu_sort(buf, hnd[perm])  # same strings, new input order
    assert np.array_equal(l3, l)
    assert oracle.certify(buf, hnd[perm], h3, l3) == (0, -1)
