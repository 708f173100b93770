"""The C-ABI library loads and exports every symbol include/s5g.h declares
(no compute calls: this runs without a GPU)."""

import re
from pathlib import Path

import pytest

from paper_1403_2056_b200 import _lib
from paper_1403_2056_b200.build import LIB_PATH, build_library

HEADER = Path(__file__).resolve().parent.parent / "include" / "s5g.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(s5g_[a-z_]+)\s*\(", text)))


def test_library_builds_and_loads():
    build_library()
    assert LIB_PATH.exists()
    L = _lib.lib()
    assert L.s5g_version() == 1


def test_every_declared_symbol_is_exported_and_bound():
    L = _lib.lib()
    names = declared_functions()
    assert "s5g_sort" in names and "s5g_sort_host" in names
    for name in names:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_workspace_is_bounded():
    L = _lib.lib()
    for n in (2, 1000, 1 << 20, 1 << 24):
        ws = L.s5g_workspace_bytes(n, 1 << 20)
        assert 32 * n < ws < 120 * n + (64 << 20)


def test_invalid_arguments_fail_without_touching_the_device():
    L = _lib.lib()
    import ctypes as C
    a = _lib.SortArgs()
    a.n = 5
    a.variant = 7
    rc = L.s5g_sort(C.byref(a))
    assert rc == _lib.S5G_E_VARIANT
    with pytest.raises(ValueError, match="unknown classify variant"):
        _lib.check(rc)
    a.variant = 0
    a.n = -1
    assert L.s5g_sort(C.byref(a)) == _lib.S5G_E_INVALID
