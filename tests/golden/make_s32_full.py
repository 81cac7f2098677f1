"""Full S^{32}_{3,8} phenotype histogram from the pinned C oracle (test fixture generator).

The reference (numba) needs ~1.4 h on 8 cores for the 2^32 genomes; the C
restatement in oracle/ is pinned to the reference by tests/test_oracle.py
(1M-slice SHA-256 digest of every output column, per-genome slices, the 1M
S32 slice histogram), so this script runs the oracle over the whole space and
commits the aggregate: hist_s32_full.json (tallies, key count, per-column
SHA-256 of the sorted records) and hist_s32_full_sample.npz (every record
whose key is 0 mod 64).
Blocks of 2^22 indices, checkpointed so an interrupted run resumes.

    python tests/golden/make_s32_full.py            # ~1 h on 8 host threads
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2205_15311_b200.classify import Histogram  # noqa: E402
from paper_2205_15311_b200.genome import space_from_preset  # noqa: E402

BLOCK = 1 << 22
KS = (7,)
HIST_K = 7
W = 6


def main() -> None:
    O.build()
    S = space_from_preset("s32_3_8")
    a, bpl, mp, mv, fp = S.kernel_args()
    n_total = S.cardinality
    ck = os.environ.get("S32_CKPT", "/tmp/s32_full.ckpt")
    acc, done = None, 0
    if os.path.exists(ck):
        acc, extra = Histogram.load(ck)
        done = int(extra["done"])
    ks = np.array(KS, np.int64)
    out = [np.zeros((BLOCK, 1), np.uint8), np.zeros(BLOCK, np.uint32), np.zeros(BLOCK, np.uint8),
           np.zeros(BLOCK, np.uint8), np.zeros(BLOCK, np.uint16), np.zeros((BLOCK, W), np.uint64)]
    t0 = time.time()
    while done < n_total:
        idx = np.arange(done, done + BLOCK, dtype=np.uint64)
        O.classify_batch(idx, a, bpl, mp, mv, fp, 19, ks, HIST_K, 0, True, *out)
        h = Histogram.from_rows(idx, *out, ks=KS, hist_k=HIST_K, W=W)
        acc = h if acc is None else acc.merge(h)
        done += BLOCK
        if (done // BLOCK) % 16 == 0 or done == n_total:
            acc.save(ck, extra=dict(done=done))
            el = time.time() - t0
            print(f"{done / n_total:7.2%}  {len(acc)} keys  {el:.0f} s", flush=True)
    finalize(acc)


def finalize(acc) -> None:
    """Compact fixtures (the full record set is ~40 MB): per-column SHA-256 of the
    sorted records (shape words [:, :5], the d=19 maximum), the tallies, and every
    record whose key is 0 mod 64 in full."""
    import hashlib
    import json

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    cols = dict(keys=acc.keys.astype(np.uint32), det=acc.det.astype(np.uint64), steric=acc.steric.astype(np.uint64),
                rep_det=acc.rep_det.astype(np.uint64), rep_any=acc.rep_any.astype(np.uint64),
                w=acc.w.astype(np.uint8), h=acc.h.astype(np.uint8), cells=acc.cells.astype(np.uint16),
                shape=np.ascontiguousarray(acc.shape[:, :5]).astype(np.uint64))
    meta = dict(space="s32_3_8", n=int(acc.tallies[0].sum()), ks=list(KS), hist_k=HIST_K, d=19, seed=0, strict=True,
                n_keys=len(acc), tallies=acc.tallies.tolist(), sha256={k: sha(v) for k, v in cols.items()},
                note="oracle/tv_oracle.c over all 2^32 indices, aggregated with classify.Histogram.from_rows")
    with open(os.path.join(HERE, "hist_s32_full.json"), "w") as f:
        json.dump(meta, f, indent=1)
    sel = (acc.keys % 64) == 0
    np.savez_compressed(os.path.join(HERE, "hist_s32_full_sample.npz"), **{k: v[sel] for k, v in cols.items()})
    print("tallies", acc.tallies.tolist(), "keys", len(acc), "sampled", int(sel.sum()))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--finalize":  # from the checkpoint of a finished run
        finalize(Histogram.load(os.environ.get("S32_CKPT", "/tmp/s32_full.ckpt"))[0])
    else:
        main()
