"""Host-side data model, mirroring strsort.strset / basecase / counters.

Same names, fields and conventions as the reference so results and inputs
interchange with it (duck-typed: any object with ``buffer``, ``handles`` and
``with_handles`` is accepted as a string set):

* ``StringSet``      strset.py:34-89  (immutable bytes buffer + int64 handles)
* ``SortedWithLcp``  basecase.py:21-33 (set, lcps with lcps[0] = -1, dchar, stats)
* ``SortStats``      counters.py:13-49
* ``from_strings``   strset.py:137-149 (contract); ``load_delimited``
  strset.py:113-134 runs on the GPU (device.load_delimited)

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
    """A set holding `strings` in order (the reference's strset.from_strings
    contract, strset.py:137-149: a string may not contain the terminator)."""
    items = [bytes(x) for x in strings]
    if any(b"\0" in x for x in items):
        raise ValueError("string contains the terminator byte")
    sizes = np.array([len(x) + 1 for x in items], dtype=np.int64)
    starts = np.concatenate(([0], np.cumsum(sizes)[:-1])).astype(np.int64) if items else sizes
    return StringSet(b"".join(x + b"\0" for x in items), starts)


def load_delimited(data: bytes, delimiter: int = 0) -> StringSet:
    """load_delimited (strset.py:113-134) with the delimiter remap and the
    string-start scan on the GPU (s5g_load_delimited); the returned set's
    buffer is the device arena copied back, its handles the device's starts.
    Same errors and output as the reference (pinned by
    tests/golden/golden_load.npz, generated from the reference itself)."""
    from . import device as D

    ds = D.load_delimited(data, delimiter)
    return StringSet(bytes(ds.arena[: ds.arena_len].cpu().numpy()), ds.handles.cpu().numpy())


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
