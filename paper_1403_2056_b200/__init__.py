"""B200-native super scalar string sample sort (S^5) with LCP array.

Drop-in for the reference's S^5 hot path (strsort 0.1.0):
``s5_sort`` (ssss.py:361-387) and ``parallel_s5`` (parallel.py:468-492),
with the same return convention (``SortedWithLcp``, lcps[0] = -1).  The
work runs in hand-written sm_100a kernels behind the C ABI in
include/s5g.h (libs5gpu.so); Python only moves buffers.
"""

from .strset import (
    LCP_UNDEF,
    WORD_CHARS,
    SortedWithLcp,
    SortStats,
    StringSet,
    from_strings,
    load_delimited,
)
from .ssss import SplitterTree, StepRecord, child_depths, s5_sort, tree_capacity
from .parallel import parallel_s5, partitioned_merge_sort
from .lcpmerge import LcpStream, binary_lcp_merge, kway_lcp_merge

__all__ = [
    "LCP_UNDEF", "LcpStream", "WORD_CHARS", "SortedWithLcp", "binary_lcp_merge", "kway_lcp_merge",
    "partitioned_merge_sort", "SortStats", "SplitterTree", "StepRecord",
    "StringSet", "child_depths", "from_strings", "load_delimited", "parallel_s5", "s5_sort",
    "tree_capacity",
]
