"""Drop-in ``parallel_s5`` (parallel.py:468-492) on GPUs.

In the reference, p is the number of forked CPU workers sharing one set.
Here the fully parallel step is the device-wide S^5 step (every CTA a
shard, bucket-major/CTA-minor offsets -- the interleaved prefix sum of
parallel.py:379-385), so one GPU already runs the reference's phased
structure.  ``p`` counts GPUs; within one process the set is sorted on the
current device.  Multi-GPU runs use one process per GPU
(``paper_1403_2056_b200.dist``: sample-sort partition + NCCL all-to-all).
"""

from __future__ import annotations

from .ssss import T_MEDIUM, s5_sort


def parallel_s5(sset, p=None, want_lcps: bool = False, want_dchar: bool = False, seed: int = 1,
                variant: str = "unroll", stats=None, t_medium: int = T_MEDIUM):
    """Sample sort on the GPU; content order matches the sequential sorter."""
    want = want_lcps or want_dchar
    return s5_sort(sset, want_lcps=want, want_dchar=want_dchar, variant=variant, seed=seed,
                   stats=stats, t_medium=t_medium)
