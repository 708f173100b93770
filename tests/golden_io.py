"""Loader for the committed golden vectors (tests/golden/golden_s5.npz)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

PATH = Path(__file__).resolve().parent / "golden" / "golden_s5.npz"


@lru_cache(maxsize=1)
def load():
    z = np.load(PATH)
    arrays = {k: z[k] for k in z.files}
    meta = json.loads(arrays.pop("meta").tobytes().decode())
    return arrays, meta


def cases():
    return sorted(load()[1]["cases"])


def case(name):
    arrays, meta = load()
    pre = name + "/"
    out = {k[len(pre):]: v for k, v in arrays.items() if k.startswith(pre)}
    out.update(meta["cases"][name])
    out["buffer_bytes"] = out["buffer"].tobytes()
    return out


def kats():
    return sorted(load()[1]["kat"])


def kat(name):
    arrays, meta = load()
    pre = name + "/"
    out = {k[len(pre):]: v for k, v in arrays.items() if k.startswith(pre)}
    out.update(meta["kat"][name])
    return out


def merges():
    return sorted(load()[1].get("merge", {}))


def merge(name):
    arrays, meta = load()
    pre = name + "/"
    out = {k[len(pre):]: v for k, v in arrays.items() if k.startswith(pre)}
    out.update(meta["merge"][name])
    return out


LOAD_PATH = Path(__file__).resolve().parent / "golden" / "golden_load.npz"


@lru_cache(maxsize=1)
def load_cases():
    """name -> {input, delimiter, error, buffer, handles}: the reference's
    load_delimited (strset.py:113-134) on seeded inputs (make_golden_load.py)."""
    z = np.load(LOAD_PATH)
    meta = json.loads(z["meta"].tobytes().decode())
    out = {}
    for name, m in meta.items():
        c = dict(m)
        c["input"] = z[f"{name}/input"]
        if m["error"] is None:
            c["buffer"] = z[f"{name}/buffer"]
            c["handles"] = z[f"{name}/handles"]
        out[name] = c
    return out
