"""Host-side data model, mirroring strsort.strset / basecase / counters.

Same names, fields and conventions as the reference so results and inputs
interchange with it (duck-typed: any object with ``buffer``, ``handles`` and
``with_handles`` is accepted as a string set):

* ``StringSet``      strset.py:34-89  (immutable bytes buffer + int64 handles)
* ``SortedWithLcp``  basecase.py:21-33 (set, lcps with lcps[0] = -1, dchar, stats)
* ``SortStats``      counters.py:13-49
* ``from_strings``   strset.py:137-149, ``load_delimited`` strset.py:113-134

Word helpers (``word_terminator_pos``, ``shared_chars``) are vectorised numpy
forms of strset.py:178-206, used on the host only to describe splitter trees
handed to a ``step_hook``.
"""

from __future__ import annotations

from dataclasses import dataclass, fields
from typing import Iterable

import numpy as np

WORD_CHARS = 8
LCP_UNDEF = -1


class StringSet:
    """Ordered handles into an immutable zero-terminated character buffer."""

    __slots__ = ("buffer", "handles", "_arr")

    def __init__(self, buffer: bytes, handles: np.ndarray):
        self.buffer = buffer
        self.handles = np.ascontiguousarray(handles, dtype=np.int64)
        self._arr = np.frombuffer(buffer, dtype=np.uint8)

    def __len__(self) -> int:
        return len(self.handles)

    @property
    def n(self) -> int:
        return len(self.handles)

    def with_handles(self, handles: np.ndarray) -> "StringSet":
        out = StringSet.__new__(StringSet)
        out.buffer = self.buffer
        out.handles = np.ascontiguousarray(handles, dtype=np.int64)
        out._arr = self._arr
        return out

    def char_array(self) -> np.ndarray:
        return self._arr

    def string_at(self, i: int) -> bytes:
        h = int(self.handles[i])
        return self.buffer[h: self.buffer.index(b"\0", h)]

    def strings(self) -> list[bytes]:
        return [self.string_at(i) for i in range(len(self))]


@dataclass
class SortStats:
    char_cmps: int = 0
    word_fetches: int = 0
    merge_buffer_cmps: int = 0
    scratch_words: int = 0
    jobs_enqueued: int = 0
    jobs_executed: int = 0
    share_events: int = 0

    def add(self, other) -> None:
        for f in fields(self):
            setattr(self, f.name, getattr(self, f.name) + getattr(other, f.name))

    def as_dict(self) -> dict[str, int]:
        return {f.name: getattr(self, f.name) for f in fields(self)}


@dataclass
class SortedWithLcp:
    set: object
    lcps: np.ndarray
    dchar: np.ndarray | None = None
    stats: object | None = None


def from_strings(strings: Iterable[bytes]) -> StringSet:
    items = list(strings)
    for s in items:
        if 0 in s:
            raise ValueError("string contains the terminator byte")
    buf = b"\0".join(items) + b"\0" if items else b""
    lens = np.fromiter((len(s) + 1 for s in items), dtype=np.int64, count=len(items))
    offs = np.zeros(len(items), dtype=np.int64)
    if len(items) > 1:
        np.cumsum(lens[:-1], out=offs[1:])
    return StringSet(buf, offs)


def load_delimited(data: bytes, delimiter: int = 0) -> StringSet:
    if not (0 <= delimiter < 256):
        raise ValueError("delimiter must be a byte value")
    if len(data) == 0:
        return StringSet(b"", np.zeros(0, dtype=np.int64))
    if delimiter != 0:
        if 0 in data:
            raise ValueError("input contains byte 0, which is reserved as terminator")
        data = data.replace(bytes([delimiter]), b"\0")
    if not data.endswith(b"\0"):
        data = data + b"\0"
    arr = np.frombuffer(data, dtype=np.uint8)
    zeros = np.flatnonzero(arr == 0)
    starts = np.empty(len(zeros), dtype=np.int64)
    starts[0] = 0
    starts[1:] = zeros[:-1] + 1
    return StringSet(data, starts)


def _be_bytes(keys: np.ndarray) -> np.ndarray:
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    return k.astype(">u8").view(np.uint8).reshape(-1, WORD_CHARS)


def word_terminator_pos(keys: np.ndarray) -> np.ndarray:
    """Characters before the first 0 byte of each word (8 if none)."""
    b = _be_bytes(keys)
    z = b == 0
    return np.where(z.any(axis=1), z.argmax(axis=1), WORD_CHARS).astype(np.int64)


def shared_chars(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Leading characters two words share, capped at the terminator."""
    ba, bb = _be_bytes(a), _be_bytes(b)
    stop = (ba != bb) | (ba == 0)
    return np.where(stop.any(axis=1), stop.argmax(axis=1), WORD_CHARS).astype(np.int64)
