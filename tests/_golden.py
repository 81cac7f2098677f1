"""Loaders for the committed reference fixtures (tests/golden/, made by make_golden.py)."""
from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
OUT_KEYS = ("cls", "hash", "w", "h", "cells", "shape")


@functools.lru_cache(None)
def vectors() -> dict:
    with open(os.path.join(GOLDEN, "vectors.json")) as f:
        return json.load(f)


@functools.lru_cache(None)
def _slices():
    return dict(np.load(os.path.join(GOLDEN, "slices.npz")))


def slice_names() -> list[str]:
    return sorted({k.split("__")[0] for k in _slices()})


def slice_case(name: str) -> dict:
    z = _slices()
    meta = json.loads(bytes(z[name + "__meta"]).decode())
    case = dict(meta)
    for k in ("idx", "mp", "mv", "free"):
        case[k] = z[f"{name}__{k}"]
    case["expected"] = {k: z[f"{name}__{k}"] for k in OUT_KEYS}
    return case


def fresh_outputs(n: int, q: int, W: int = 6, prefill: int = 0) -> dict:
    return dict(cls=np.zeros((n, q), np.uint8), hash=np.zeros(n, np.uint32), w=np.zeros(n, np.uint8),
                h=np.zeros(n, np.uint8), cells=np.zeros(n, np.uint16),
                shape=np.full((n, W), prefill, np.uint64))


def digests() -> dict:
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        return json.load(f)


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def hist_golden(name: str) -> dict:
    return dict(np.load(os.path.join(GOLDEN, f"hist_{name}.npz")))


def histogram_from_outputs(out: dict, idx: np.ndarray, ks, hist_k) -> dict:
    """Aggregate per-genome classify_batch outputs exactly as make_golden.histogram does."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_mg", os.path.join(GOLDEN, "make_golden.py"))
    # make_golden imports the reference at module import time; replicate its histogram here instead
    q = list(ks).index(hist_k)
    hc = out["cls"][:, q]
    tallies = np.zeros((len(ks), 5), np.int64)
    for j in range(len(ks)):
        c = out["cls"][:, j]
        for v, col in ((0, 0), (1, 1), (2, 2), (3, 3), (255, 4)):
            tallies[j, col] = int((c == v).sum())
    sel = (hc == 0) | (hc == 2)
    hs = out["hash"][sel]
    ii = idx[sel]
    isdet = hc[sel] == 0
    keys, inv = np.unique(hs, return_inverse=True)
    U = keys.shape[0]
    det = np.bincount(inv, weights=isdet, minlength=U).astype(np.int64)
    ste = np.bincount(inv, weights=~isdet, minlength=U).astype(np.int64)
    BIG = np.iinfo(np.uint64).max
    rep_det = np.full(U, BIG, np.uint64)
    rep_any = np.full(U, BIG, np.uint64)
    np.minimum.at(rep_any, inv, ii)
    np.minimum.at(rep_det, inv[isdet], ii[isdet])
    del spec
    return dict(keys=keys, det=det, steric=ste, rep_det=rep_det, rep_any=rep_any, tallies=tallies)


def s32_sample(kind: str) -> tuple[np.ndarray, dict]:
    """Indices and reference digests of the reference-pinned S32 samples
    (tests/golden/make_s32_sample.py): 'blocks' = bench.py's 64 x 2^16 blocks,
    'random' = 2^22 uniformly random indices (unique, sorted)."""
    with open(os.path.join(GOLDEN, "s32_sample_digests.json")) as f:
        meta = json.load(f)[kind]
    if kind == "blocks":
        s = meta["sample"]
        idx = (np.arange(s["blocks"], dtype=np.uint64)[:, None] * np.uint64(s["stride"])
               + np.arange(s["block"], dtype=np.uint64)[None, :]).reshape(-1)
    else:
        idx = np.unique(np.random.default_rng(32).integers(0, 1 << 32, 1 << 22, dtype=np.uint64))
        assert idx.shape[0] == meta["sample"]["n"]
    return idx, meta
