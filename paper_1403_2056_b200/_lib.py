"""ctypes binding of libs5gpu.so (include/s5g.h).

The library is the product: there is no fallback.  Loading fails loudly
when the shared object is missing; calls fail loudly without a CUDA device.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .build import LIB_PATH

_i64, _u64, _i32, _p = C.c_int64, C.c_uint64, C.c_int32, C.c_void_p

S5G_OK = 0
S5G_E_INVALID = -1
S5G_E_VARIANT = -2
S5G_E_CUDA = -3
S5G_E_WORKSPACE = -4
S5G_E_NCCL = -5
S5G_ARENA_PAD = 16
VARIANTS = {"unroll": 0, "equal": 1}

STATS_FIELDS = (
    "char_cmps", "word_fetches", "merge_buffer_cmps", "scratch_words",
    "jobs_enqueued", "jobs_executed", "share_events",
)


class Stats(C.Structure):
    _fields_ = [(f, C.c_int64) for f in STATS_FIELDS]


STEP_CB = C.CFUNCTYPE(None, _p, _i64, _i64, _i64, _i64, C.POINTER(_i64), C.POINTER(_u64))


class SortArgs(C.Structure):
    _fields_ = [
        ("arena", _p), ("arena_len", _i64), ("handles", _p), ("n", _i64), ("depth", _i64),
        ("out_handles", _p), ("out_lcps", _p), ("out_dchar", _p),
        ("workspace", _p), ("workspace_bytes", C.c_size_t), ("stream", _p),
        ("variant", _i32), ("v", _i32), ("seed", _u64), ("t_medium", _i64),
        ("stats", C.POINTER(Stats)), ("step_cb", STEP_CB), ("step_ctx", _p),
    ]


class MultiArgs(C.Structure):
    _fields_ = [
        ("arena", _p), ("arena_len", _i64), ("handles", _p), ("n", _i64), ("depth", _i64),
        ("out_handles", _p), ("out_lcps", _p), ("out_dchar", _p),
        ("num_devices", _i32), ("device_ids", C.POINTER(_i32)),
        ("variant", _i32), ("v", _i32), ("seed", _u64), ("t_medium", _i64),
        ("stats", C.POINTER(Stats)),
    ]


class KernelProfile(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("units", C.c_int64),
                ("ms", C.c_double), ("bytes", C.c_int64)]


# every symbol include/s5g.h declares, with its signature
SIGNATURES = {
    "s5g_sort": (C.c_int, [C.POINTER(SortArgs)]),
    "s5g_workspace_bytes": (C.c_size_t, [_i64, _i64]),
    "s5g_sort_host": (C.c_int, [_p, _i64, _p, _i64, _i64, _p, _p, _p, _i32, _i32, _u64, _i64,
                                C.POINTER(Stats)]),
    "s5g_release_cached_memory": (None, []),
    "s5g_sort_multi": (C.c_int, [C.POINTER(MultiArgs)]),
    "s5g_extract_keys": (C.c_int, [_p, _i64, _p, _i64, _i64, _p, _p]),
    "s5g_select_splitters": (C.c_int, [_p, _i64, _i64, _p, _p, _p, _p, _p]),
    "s5g_classify": (C.c_int, [_p, _i64, _p, _p, _i64, _i32, _p, _p]),
    "s5g_fill_dchar": (C.c_int, [_p, _p, _p, _i64, _p, _p]),
    "s5g_partition": (C.c_int, [_p, _i64, _p, _i64, _i64, _p, _p, _p, _p, _i32, _p, _p]),
    "s5g_lengths": (C.c_int, [_p, _i64, _p, _i64, _p, _p]),
    "s5g_load_delimited": (C.c_int, [_p, _i64, _i32, _p, C.POINTER(_i64), _p, C.c_size_t, _p]),
    "s5g_load_delimited_n": (C.c_int, [_p, _i64, _i32, _p, _i64, C.POINTER(_i64), _p, C.c_size_t, _p]),
    "s5g_load_delimited_rank": (C.c_int, [_p, _i64, _i32, _p, _i64, C.POINTER(_i64), _p, _p, C.c_size_t, _p]),
    "s5g_rank_positions": (C.c_int, [_p, _i64, _p, _p, _i64, _p, _p]),
    "s5g_dist_stats": (C.c_int, [_p, _i64, C.POINTER(_i64), C.POINTER(_i64), _p]),
    "s5g_pack": (C.c_int, [_p, _i64, _p, _p, _p, _i64, _p, _p]),
    "s5g_profile_enable": (None, [C.c_int]),
    "s5g_profile_reset": (None, []),
    "s5g_profile_read": (C.c_int, [C.POINTER(KernelProfile), C.c_int]),
    "s5g_profile_timeline": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int]),
    "s5g_launch_count": (C.c_ulonglong, []),
    "s5g_set_l2_fetch_granularity": (None, [C.c_int]),
    "s5g_finisher_counters": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int, C.c_int]),
    "s5g_merge_workspace_bytes": (C.c_size_t, [_i64, _i32]),
    "s5g_group_workspace_bytes": (C.c_size_t, [_i64, _i32]),
    "s5g_group_by_dest": (C.c_int, [_p, _i64, _i32, _p, _p, _p, C.c_size_t, _p]),
    "s5g_positions": (C.c_int, [_p, _i64, _p, _i64, _p, _i64, _p, _p]),
    "s5g_input_positions_workspace_bytes": (C.c_size_t, [_i64]),
    "s5g_input_positions": (C.c_int, [_p, _p, _i64, _i64, _p, _p, C.c_size_t, _p]),
    "s5g_gather_i64": (C.c_int, [_p, _p, _i64, _p, _p]),
    "s5g_pack_plan_workspace_bytes": (C.c_size_t, [_i64]),
    "s5g_pack_plan": (C.c_int, [_p, _i64, _p, _p, _i64, _p, _i32, _p, _p, _p, _p, C.c_size_t, _p]),
    "s5g_kway_merge": (C.c_int, [_p, _i64, _i32, C.POINTER(_i64), _p, _p, _p, _i64, _p, _p, _p,
                                 C.c_size_t, _p, C.POINTER(Stats)]),
    "s5g_last_error": (C.c_char_p, []),
    "s5g_version": (C.c_int, []),
}


class S5GError(RuntimeError):
    pass


_lib = None


def lib(path: Path | None = None):
    global _lib
    if _lib is None:
        import os

        # S5G_LIB: an alternative build of the same library (A/B tuning runs)
        p = Path(path) if path else Path(os.environ.get("S5G_LIB") or LIB_PATH)
        if not p.exists():
            raise ImportError(
                f"{p} is missing: build it with `python -m paper_1403_2056_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == S5G_OK:
        return
    msg = lib().s5g_last_error().decode(errors="replace")
    if rc in (S5G_E_INVALID, S5G_E_VARIANT):
        raise ValueError(msg)
    raise S5GError(f"s5g error {rc}: {msg}")


def profile(enable: bool | None = None, reset: bool = False, serial: bool = False) -> dict[str, dict]:
    """Per-kernel event timings collected by the library.  serial: every kernel
    on the caller's stream, so each launch's time is exclusive."""
    L = lib()
    if reset:
        L.s5g_profile_reset()
    if enable is not None:
        L.s5g_profile_enable((2 if serial else 1) if enable else 0)
    buf = (KernelProfile * 32)()
    k = L.s5g_profile_read(buf, 32)
    return {buf[i].name.decode(): {"launches": int(buf[i].launches), "units": int(buf[i].units),
                                   "ms": float(buf[i].ms),
                                   "bytes": int(buf[i].bytes)} for i in range(k)}


def timeline() -> list[tuple[str, int, float, float]]:
    """(kernel, stream, start ms, end ms) of every launch of the last profiled sort."""
    L = lib()
    names = list(profile().keys())
    cap = 4096
    kid = (C.c_int * cap)()
    sid = (C.c_int * cap)()
    t0 = (C.c_float * cap)()
    t1 = (C.c_float * cap)()
    k = min(cap, L.s5g_profile_timeline(kid, sid, t0, t1, cap))
    return [(names[kid[i]], int(sid[i]), float(t0[i]), float(t1[i])) for i in range(k)]


def finisher_counters(reset: bool = False) -> dict[str, dict[str, int]]:
    """CTAs / rounds / two-word rounds / group-mode exits per k_cta_sort<W>."""
    buf = (C.c_ulonglong * 12)()
    check(lib().s5g_finisher_counters(buf, 12, 1 if reset else 0))
    return {f"k_cta_sort<{W}>": {"ctas": buf[4 * c], "rounds": buf[4 * c + 1],
                                  "two_word": buf[4 * c + 2], "group_mode": buf[4 * c + 3]}
            for c, W in enumerate((2, 4, 8))}


def launch_count() -> int:
    return int(lib().s5g_launch_count())
