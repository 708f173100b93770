"""Registration with the reference harness's plugin API
(``strsort.bench.register_algorithm``, bench.py:151-152)."""

from __future__ import annotations

from .parallel import parallel_s5
from .ssss import s5_sort


def _algo_gpu_s5(sset, threads, seed, stats):
    return s5_sort(sset, seed=seed, stats=stats)


def _algo_gpu_ps5(sset, threads, seed, stats):
    # the harness's worker count becomes the GPU count, capped at the visible
    # devices (parallel_s5's p counts GPUs)
    from .parallel import visible_devices

    return parallel_s5(sset, p=max(1, min(int(threads or 1), visible_devices())), seed=seed,
                       stats=stats)


def register_with_strsort() -> bool:
    """Register ``gpu-s5`` and ``gpu-ps5``; False when strsort is absent."""
    try:
        import strsort.bench as B
    except ImportError:
        return False
    B.register_algorithm("gpu-s5", _algo_gpu_s5)
    B.register_algorithm("gpu-ps5", _algo_gpu_ps5)
    return True
