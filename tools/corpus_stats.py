"""Achieved statistics of a corpus: duplicate fraction
(1 - distinct/n), L/n (mean LCP of the sorted order), D/n, average length --
computed with the CPU oracle.  usage: python tools/corpus_stats.py CFG [SCALE] [k=v ...]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_1403_2056_b200 import corpora  # noqa: E402


def stats(buf, hnd):
    h, l, _ = oracle.parallel_s5(buf, hnd)
    lens = oracle.lengths(buf, h)
    D, L, avg = oracle.dist_stats(buf, h, l)
    dup = int(((l[1:] == lens[1:]) & (lens[1:] == lens[:-1])).sum())
    n = len(hnd)
    return {"n": n, "dup_frac": dup / n, "L_per_n": L / n, "D_per_n": D / n, "avg_len": avg,
            "N_bytes": int(len(buf))}


if __name__ == "__main__":
    cfg = sys.argv[1]
    scale = float(sys.argv[2]) if len(sys.argv) > 2 and "=" not in sys.argv[2] else 1.0
    kw = dict(a.split("=") for a in sys.argv[2:] if "=" in a)
    kw = {k: (float(v) if "." in v else int(v)) for k, v in kw.items()}
    if kw:
        fn = {"c3_urls": corpora.gen_urls}[cfg]
        buf, hnd = fn(int((1 << 23) * scale), 2, **kw)
    else:
        buf, hnd = corpora.CONFIGS[cfg](scale)
    print(cfg, scale, kw, {k: round(v, 4) if isinstance(v, float) else v for k, v in stats(buf, hnd).items()})
