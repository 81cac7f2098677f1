"""Full S^{32}_{3,8} phenotype histogram from the pinned C oracle (test fixture generator).

The reference (numba) needs ~1.4 h on 8 cores for the 2^32 genomes; the C
restatement in oracle/ is pinned to the reference by tests/test_oracle.py
(1M-slice SHA-256 digest of every output column, per-genome slices, the 1M
S32 slice histogram), so this script runs the oracle over the whole space and
commits the aggregate: hist_s32_full.npz (every record + per-k tallies).
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
    np.savez_compressed(os.path.join(HERE, "hist_s32_full.npz"), keys=acc.keys, det=acc.det, steric=acc.steric,
                        rep_det=acc.rep_det, rep_any=acc.rep_any, w=acc.w, h=acc.h, cells=acc.cells,
                        shape=acc.shape, tallies=acc.tallies)
    print("tallies", acc.tallies.tolist(), "keys", len(acc))


if __name__ == "__main__":
    main()
