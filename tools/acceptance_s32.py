"""SPEC ACCEPTANCE 6 (S^{32}_{3,8}) on the device, in full-run mode.

  * the whole space (2^32 genomes, k = 7, d = 19, seed 0): number of deterministic shapes
    (hashes with DET genomes), reported against the paper's 361;
  * a uniform random 2^24-genome sample: its most frequent deterministic shapes must
    all be S_{2,8} shapes ("building blocks", SPEC section 4.3);
  * the tile-2-inert slice (s32_3_8_inert2): every deterministic shape is an S_{2,8} one
    (also asserted by tests/test_gpu_api.py).

usage: python tools/acceptance_s32.py [out.json] [top]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2205_15311_b200.classify import DeviceHistogram, enumerate_space, shape_words_for  # noqa: E402
from paper_2205_15311_b200.genome import SearchSpace, space_from_preset  # noqa: E402


def run(top: int = 20) -> dict:
    s28 = enumerate_space(SearchSpace(2, 8), d=19, ks=(8,), batch_size=1 << 24)
    det28 = set(s28.keys[s28.det > 0].tolist())
    any28 = set(s28.keys.tolist())  # DET or STERIC-attributed S_{2,8} shapes
    S32 = space_from_preset("s32_3_8")
    t0 = time.time()
    full = enumerate_space(S32, d=19, ks=(7,), batch_size=1 << 30, capacity=1 << 21)
    t_full = time.time() - t0
    det32 = full.keys[full.det > 0]
    rng = np.random.default_rng(2205)
    idx = np.unique(rng.integers(0, 1 << 32, 1 << 24, dtype=np.uint64))
    dh = DeviceHistogram((7,), 7, shape_words_for(19), 1 << 20)
    dh.enumerate_indices(S32, idx, 19, 0, True)
    smp = dh.export()
    dh.close()
    order = np.argsort(-smp.det.astype(np.int64), kind="stable")
    top_keys = [int(smp.keys[i]) for i in order[:top] if smp.det[i] > 0]
    inert = enumerate_space(space_from_preset("s32_3_8_inert2"), d=19, ks=(7,), batch_size=1 << 20)
    det_inert = set(inert.keys[inert.det > 0].tolist())
    return {
        "full_space": {"genomes": int(full.tallies[0].sum()), "phenotype_hashes": len(full),
                       "deterministic_shapes": int(det32.size), "paper_deterministic_shapes": 361,
                       "tallies_k7": dict(zip(("det", "trivial", "steric", "unbound", "error"),
                                              map(int, full.tallies[0]))), "seconds": t_full},
        "sample": {"genomes": int(idx.size), "seed": 2205, "top": top,
                   "top_det_shapes_in_s28": sum(k in det28 for k in top_keys), "top_det_shapes": len(top_keys),
                   "top_det_cells": [int(smp.cells[i]) for i in order[:top] if smp.det[i] > 0]},
        "inert2_slice": {"deterministic_shapes": len(det_inert), "all_in_s28_shapes": det_inert <= any28,
                         "in_s28_det_shapes": len(det_inert & det28),
                         "note": "S32 uses k = 7, S28 k = 8: a shape DET at k = 7 can be STERIC-attributed at k = 8"},
        "s28_deterministic_shapes": len(det28),
    }


if __name__ == "__main__":
    res = run(int(sys.argv[2]) if len(sys.argv) > 2 else 20)
    txt = json.dumps(res, indent=1)
    print(txt)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(txt + "\n")
