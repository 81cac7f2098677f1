"""Generate golden fixtures by running the REFERENCE (tilevolve, numba) in the
build container.  /root/reference is not present on the GPU box, so the
outputs are committed under tests/golden/ and this script is the recipe.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs:
  vectors.json        oat hashes, RNG streams, classify_single / assemble_single cases
  slices.npz          per-genome classify_batch outputs on small index slices
  hist_<name>.npz     phenotype histograms + class tallies on large ranges
  digests.json        SHA-256 of reference classify_batch outputs on large ranges
"""
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


def space_args(space):
    free = np.array(space.free_positions(), np.int64)
    mp = np.array([p for p, _ in space.fixed_mask], np.int64)
    mv = np.array([v for _, v in space.fixed_mask], np.uint8)
    return mp, mv, free


def run_batch(space, idx, ks, hist_k, seed=0, strict=True, d=19, prefill=0, workers=8, batch=1 << 16):
    n = idx.shape[0]
    q = len(ks)
    mp, mv, free = space_args(space)
    ksa = np.array(ks, np.int64)
    out = dict(cls=np.zeros((n, q), np.uint8), hash=np.zeros(n, np.uint32), w=np.zeros(n, np.uint8),
               h=np.zeros(n, np.uint8), cells=np.zeros(n, np.uint16), shape=np.full((n, W), prefill, np.uint64))

    def work(s):
        e = min(n, s + batch)
        K.classify_batch(idx[s:e], space.a, space.bits_per_label, mp, mv, free, d, ksa, hist_k,
                         np.uint64(seed), strict, out["cls"][s:e], out["hash"][s:e], out["w"][s:e],
                         out["h"][s:e], out["cells"][s:e], out["shape"][s:e])
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(work, range(0, n, batch)))
    return out


def histogram(out, idx, ks, hist_k):
    """Phenotype histogram (SPEC classify:235-240, 297-306): per hash det/steric
    counts, lowest DET index, lowest DET-or-STERIC index, payload."""
    q = ks.index(hist_k)
    hc = out["cls"][:, q]
    tallies = np.zeros((len(ks), 5), np.int64)  # DET TRIV STERIC UNB ERROR
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
    # payload is a function of the hash: take the first occurrence, assert consistency
    first = np.full(U, -1, np.int64)
    pos = np.nonzero(sel)[0]
    order = np.argsort(inv, kind="stable")
    first[inv[order][::-1]] = pos[order][::-1]
    w = out["w"][first]; h = out["h"][first]; cells = out["cells"][first]; shape = out["shape"][first]
    chk = (out["w"][pos] == w[inv]) & (out["h"][pos] == h[inv]) & (out["cells"][pos] == cells[inv]) & \
        np.all(out["shape"][pos] == shape[inv], axis=1)
    assert chk.all(), "hash collision between distinct payloads"
    return dict(keys=keys, det=det, steric=ste, rep_det=rep_det, rep_any=rep_any, w=w, h=h, cells=cells,
                shape=shape, tallies=tallies)


def digests(out):
    return {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in out.items()}


def edges_of(tiles):
    lab = np.array([v for t in tiles for v in t], np.uint8)
    return K.edges_from_labels(lab, len(tiles))


def main():
    t0 = time.time()
    rng = np.random.default_rng(20250517)
    S28 = G.SearchSpace(2, 8)
    S32 = G.space_from_preset("s32_3_8")
    vec = {}

    # --- OAT hash (_k:79-85)
    oat = [[], [0x61], [1, 2, 3], [1, 1, 0, 0], [1, 2, 0, 0, 0, 1], [2, 1, 0, 0, 1, 0]]
    for _ in range(32):
        oat.append([int(x) for x in rng.integers(0, 256, int(rng.integers(0, 64)))])
    vec["oat"] = [[b, int(K.oat_hash_bytes(np.array(b, np.uint8)))] for b in oat]

    # --- RNG streams (_k:45-60)
    streams = []
    for seed, idx, run in [(0, 0, 0), (0, 0x800000, 3), (12345, 0x9E370000, 6), (2**64 - 1, 2**40 + 7, 31)]:
        rs = np.array([K._stream_state(np.uint64(seed), np.uint64(idx), run)], np.uint64)
        draws = [int(K._rng_next(rs)) for _ in range(16)]
        rs2 = np.array([K._stream_state(np.uint64(seed), np.uint64(idx), run)], np.uint64)
        below = [int(K._rng_below(rs2, n)) for n in (2, 3, 4, 2, 3, 4, 5, 7)]
        streams.append(dict(seed=seed, idx=idx, run=run, draws=[str(x) for x in draws], below=below))
    vec["streams"] = streams

    # --- classify_single (_k:471-484)
    tilesets = [((0, 0, 0, 0), (0, 0, 0, 0)), ((2, 0, 0, 0), (0, 0, 1, 0)), ((2, 0, 1, 0), (0, 0, 0, 0)),
                ((1, 1, 1, 1), (2, 0, 0, 0)), ((1, 1, 1, 1), (2, 2, 2, 2)), ((7, 0, 0, 0), (7, 0, 0, 0)),
                ((1, 0, 0, 0), (0, 0, 0, 0))]
    for _ in range(40):
        a = int(rng.integers(1, 4))
        tilesets.append(tuple(tuple(int(x) for x in rng.integers(0, 8, 4)) for _ in range(a)))
    # genomes that are steric/det in S28 at k=8 (found from the slice below)
    cases = []
    for ti, ts in enumerate(tilesets):
        for (d, k, seed, strict) in [(19, 8, 0, True), (19, 1, 0, True), (19, 16, 7, True), (11, 8, 0, True),
                                     (19, 8, 0, False), (21, 4, 3, True)]:
            if ti >= 7 and (d, k) not in [(19, 8), (11, 8)]:
                continue
            edges = edges_of(ts)
            sw = np.full((d * d + 63) // 64, 0xAB, np.uint64)
            gi = ti * 1000 + 17
            st, cls, hs, w, h, nc = K.classify_single(edges, len(ts), d, k, np.uint64(seed), np.uint64(gi), strict, sw)
            cases.append(dict(tiles=ts, d=d, k=k, seed=seed, strict=strict, genome_index=gi,
                              result=[int(st), int(cls), int(hs), int(w), int(h), int(nc)],
                              shape=[str(int(x)) for x in sw]))
    vec["classify_single"] = cases

    # --- assemble_single (_k:455-468)
    asm = []
    for ti, ts in enumerate(tilesets[:20]):
        for run in (0, 1, 5):
            d = 19 if run != 5 else 9
            edges = edges_of(ts)
            g = np.empty(d * d, np.int16)
            res = K.assemble_single(edges, len(ts), d, np.uint64(0), np.uint64(ti), run, True, g)
            asm.append(dict(tiles=ts, d=d, run=run, genome_index=ti, result=[int(x) for x in res],
                            grid=[int(x) for x in g]))
    vec["assemble_single"] = asm
    with open(os.path.join(HERE, "vectors.json"), "w") as f:
        json.dump(vec, f)
    print("vectors", time.time() - t0)

    # --- per-genome slices
    sl = {}
    def add(name, space, idx, ks, hist_k, **kw):
        out = run_batch(space, idx.astype(np.uint64), ks, hist_k, **kw)
        mp, mv, free = space_args(space)
        meta = dict(a=space.a, bpl=space.bits_per_label, ks=list(ks), hist_k=hist_k,
                    seed=kw.get("seed", 0), strict=kw.get("strict", True), d=kw.get("d", 19),
                    prefill=kw.get("prefill", 0))
        sl[name + "__idx"] = idx.astype(np.uint64)
        sl[name + "__mp"] = mp
        sl[name + "__mv"] = mv
        sl[name + "__free"] = free
        sl[name + "__meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
        for k, v in out.items():
            sl[name + "__" + k] = v
    add("s28_800000", S28, np.arange(0x800000, 0x800000 + 4096), (1, 2, 4, 8), 8)
    add("s28_0", S28, np.arange(0, 4096), (1, 2, 4, 8), 8)
    add("s28_rand", S28, rng.integers(0, 1 << 24, 8192), (1, 2, 4, 8), 8)
    add("s28_rand_prefill", S28, rng.integers(0, 1 << 24, 2048), (1, 2, 4, 8), 8, prefill=0xABABABABABABABAB)
    add("s28_rand_nonstrict", S28, rng.integers(0, 1 << 24, 4096), (1, 2, 4, 8), 8, strict=False)
    add("s28_rand_seed", S28, rng.integers(0, 1 << 24, 4096), (1, 2, 4, 8), 8, seed=12345)
    add("s28_rand_hk4", S28, rng.integers(0, 1 << 24, 4096), (1, 2, 4, 8), 4)
    add("s28_rand_k32", S28, rng.integers(0, 1 << 24, 1024), (1, 2, 4, 8, 16, 32), 32)
    add("s28_rand_d21", S28, rng.integers(0, 1 << 24, 2048), (1, 2, 4, 8), 8, d=21)
    add("s28_rand_d11", S28, rng.integers(0, 1 << 24, 2048), (1, 2, 4, 8), 8, d=11)
    add("s28_rand_d5", S28, rng.integers(0, 1 << 24, 1024), (1, 8), 8, d=5)
    add("s28_rand_d3", S28, rng.integers(0, 1 << 24, 1024), (8,), 8, d=3)
    add("s28_rand_d31", S28, rng.integers(0, 1 << 24, 1024), (1, 2, 4, 8), 8, d=31)
    add("s32_9e37", S32, np.arange(0x9E370000, 0x9E370000 + 4096), (7,), 7)
    add("s32_rand", S32, rng.integers(0, 1 << 32, 8192, dtype=np.uint64), (7,), 7)
    add("s32i2_rand", G.space_from_preset("s32_3_8_inert2"), rng.integers(0, 1 << 20, 2048), (1, 7), 7)
    add("s24_full", G.SearchSpace(2, 4), np.arange(0, 1 << 16), (1, 2, 4, 8, 16), 16)
    add("s18_full", G.SearchSpace(1, 8), np.arange(0, 1 << 12), (1, 8), 8)
    add("s34_rand", G.SearchSpace(3, 4), rng.integers(0, 1 << 24, 2048), (1, 8), 8)
    add("s48_rand", G.SearchSpace(4, 8), rng.integers(0, 1 << 48, 2048, dtype=np.uint64), (1, 8), 8)
    add("s216_rand", G.SearchSpace(2, 16), rng.integers(0, 1 << 32, 2048, dtype=np.uint64), (1, 8), 8)
    add("s12_rand", G.SearchSpace(1, 2), np.arange(0, 16), (1, 8), 8)
    np.savez_compressed(os.path.join(HERE, "slices.npz"), **sl)
    print("slices", time.time() - t0)

    # --- large ranges: histograms + digests
    dig = {}
    for name, space, start, n, ks in [("s28_1m", S28, 0x800000, 1 << 20, (1, 2, 4, 8)),
                                      ("s32_1m", S32, 0x9E370000, 1 << 20, (7,)),
                                      ("s28_full", S28, 0, 1 << 24, (1, 2, 4, 8))]:
        idx = np.arange(start, start + n, dtype=np.uint64)
        out = run_batch(space, idx, ks, ks[-1])
        dig[name] = dict(start=start, n=n, ks=list(ks), digests=digests(out))
        hh = histogram(out, idx, list(ks), ks[-1])
        np.savez_compressed(os.path.join(HERE, f"hist_{name}.npz"), **hh)
        print(name, hh["tallies"].tolist(), "keys", hh["keys"].shape[0], time.time() - t0)
        del out
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(dig, f, indent=1)


if __name__ == "__main__":
    main()
