"""Golden vectors for the input side: the REFERENCE's own
strsort.strset.load_delimited (strset.py:113-134), run in the build container
(/root/reference/pkg/src), on seeded inputs.  Output: golden_load.npz with,
per case, the raw input bytes, the delimiter, and the reference's buffer and
handles -- or the ValueError message it raised.  The GPU path
(s5g_load_delimited) is checked against these in tests/test_gpu_extras.py.

Usage:  python tests/golden/make_golden_load.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden_load.npz"


def cases() -> dict[str, tuple[bytes, int]]:
    rng = np.random.default_rng(77)
    out = {
        "nul_two": (b"a\0b\0", 0), "nl_trailing": (b"ab\ncd\n", 10), "nl_open": (b"ab\ncd", 10),
        "empty": (b"", 10), "only_delims": (b"\n\n", 10), "one_char": (b"x", 0),
        "nul_empty_mid": (b"abc\0\0d", 0), "zero_with_delim": (b"a\0b\n", 10),
        "tab_high_bytes": (bytes([9, 200, 255, 9, 1, 2, 9]), 9), "delim_255": (b"ab\xffcd\xff\xff", 255),
        "single_delim": (b"\n", 10), "empty_nul": (b"\0", 0),
    }
    lines = [bytes(rng.integers(97, 123, size=int(rng.integers(0, 30)), dtype=np.uint8))
             for _ in range(20000)]
    out["lines_20000"] = (b"\n".join(lines), 10)
    out["lines_20000_trailing"] = (b"\n".join(lines[:5000]) + b"\n", 10)
    chunk = bytes(rng.integers(1, 256, size=70000, dtype=np.uint8))  # bytes 1..255, delim 7
    out["binary_70000"] = (chunk, 7)
    return out


def main() -> None:
    sys.path.insert(0, str(REF))
    from strsort.strset import load_delimited

    arrays, meta = {}, {}
    for name, (data, delim) in cases().items():
        arrays[f"{name}/input"] = np.frombuffer(data, dtype=np.uint8).copy()
        try:
            s = load_delimited(data, delim)
            arrays[f"{name}/buffer"] = np.frombuffer(s.buffer, dtype=np.uint8).copy()
            arrays[f"{name}/handles"] = np.asarray(s.handles, dtype=np.int64)
            meta[name] = {"delimiter": delim, "error": None}
        except ValueError as e:
            meta[name] = {"delimiter": delim, "error": str(e)}
    arrays["meta"] = np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({len(meta)} cases)")


if __name__ == "__main__":
    main()
