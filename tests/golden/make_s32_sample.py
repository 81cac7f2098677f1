"""Reference-pinned S^{32}_{3,8} golden at scale: run the REFERENCE (tilevolve, numba,
/root/reference/pkg/src/tilevolve/_kernels.py:404-452) over the 64 evenly spaced blocks of
2^16 consecutive indices that bench.py's S32 CPU baseline uses (4,194,304 genomes spread
over the whole 2^32 index range: every seed-tile label combination's high bits), and
commit the SHA-256 of every per-genome output array plus the phenotype histogram; and
the same for 2^22 uniformly random indices (sorted, numpy seed 32), whose phenotypes are
far more varied than the blocks' (the blocks only vary the low index bits).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_s32_sample.py

Outputs: s32_sample_digests.json, hist_s32_{blocks,random}.npz.  The histogram payload of a key
is the row of its lowest-index genome (collisions between distinct shapes under one
32-bit hash resolve exactly as the per-genome aggregation in index order does)."""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from tilevolve import _kernels as K  # noqa: E402
from tilevolve import genome as G  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
W = 6
BLOCKS, BLOCK = 64, 1 << 16


def sample_indices(kind: str) -> np.ndarray:
    if kind == "blocks":
        return (np.arange(BLOCKS, dtype=np.uint64)[:, None] * np.uint64((1 << 32) // BLOCKS)
                + np.arange(BLOCK, dtype=np.uint64)[None, :]).reshape(-1)
    return np.unique(np.random.default_rng(32).integers(0, 1 << 32, 1 << 22, dtype=np.uint64))


def main():
    res = {}
    for kind in ("blocks", "random"):
        res[kind] = run(kind)
    with open(os.path.join(HERE, "s32_sample_digests.json"), "w") as f:
        json.dump(res, f, indent=1)


def run(kind):
    t0 = time.time()
    space = G.space_from_preset("s32_3_8")
    free = np.array(space.free_positions(), np.int64)
    mp = np.array([p for p, _ in space.fixed_mask], np.int64)
    mv = np.array([v for _, v in space.fixed_mask], np.uint8)
    idx = sample_indices(kind)
    n = idx.shape[0]
    ks = np.array([7], np.int64)
    out = dict(cls=np.zeros((n, 1), np.uint8), hash=np.zeros(n, np.uint32), w=np.zeros(n, np.uint8),
               h=np.zeros(n, np.uint8), cells=np.zeros(n, np.uint16), shape=np.zeros((n, W), np.uint64))

    def work(s):
        e = min(n, s + BLOCK)
        K.classify_batch(idx[s:e], space.a, space.bits_per_label, mp, mv, free, 19, ks, 7, np.uint64(0), True,
                         out["cls"][s:e], out["hash"][s:e], out["w"][s:e], out["h"][s:e], out["cells"][s:e],
                         out["shape"][s:e])
    with ThreadPoolExecutor(os.cpu_count() or 8) as ex:
        list(ex.map(work, range(0, n, BLOCK)))
    print("reference classify_batch", n, "genomes", round(time.time() - t0, 1), "s")
    dig = {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in out.items()}
    c = out["cls"][:, 0]
    tallies = [[int((c == v).sum()) for v in (0, 1, 2, 3, 255)]]
    sel = np.nonzero((c == 0) | (c == 2))[0]
    keys, inv = np.unique(out["hash"][sel], return_inverse=True)
    U = keys.shape[0]
    isdet = c[sel] == 0
    big = np.iinfo(np.uint64).max
    rep_any = np.full(U, big, np.uint64)
    rep_det = np.full(U, big, np.uint64)
    np.minimum.at(rep_any, inv, idx[sel])
    np.minimum.at(rep_det, inv[isdet], idx[sel][isdet])
    first = sel[np.lexsort((idx[sel], inv))][np.r_[0, np.flatnonzero(np.diff(np.sort(inv))) + 1]]
    assert np.array_equal(idx[first], rep_any)
    hist = dict(keys=keys.astype(np.uint32), det=np.bincount(inv, isdet, U).astype(np.uint64),
                steric=np.bincount(inv, ~isdet, U).astype(np.uint64), rep_det=rep_det, rep_any=rep_any,
                w=out["w"][first], h=out["h"][first], cells=out["cells"][first], shape=out["shape"][first, :5],
                tallies=np.array(tallies, np.int64))
    np.savez_compressed(os.path.join(HERE, f"hist_s32_{kind}.npz"), **hist)
    print(kind, "tallies", tallies, "keys", U, round(time.time() - t0, 1), "s")
    sample = (dict(blocks=BLOCKS, block=BLOCK, stride=(1 << 32) // BLOCKS) if kind == "blocks"
              else dict(n=int(n), rng="numpy default_rng(32).integers(0, 2^32, 2^22, uint64), unique, sorted"))
    return dict(sample=sample, ks=[7], hist_k=7, d=19, seed=0, strict=True, W=W,
                generator="reference tilevolve._kernels.classify_batch (numba)", digests=dig, tallies=tallies,
                n_keys=int(U))


if __name__ == "__main__":
    main()
