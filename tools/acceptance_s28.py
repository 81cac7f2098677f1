"""SPEC ACCEPTANCE 2 (S_{2,8} reproduction) on the device.

Full S_{2,8} at d=19, seed 0, strict contacts, prefix ks = (1, 2, 4, 8, 16, 32),
hash attribution at k = 8:
  (a) hashes carrying both DETERMINISTIC and STERIC genomes (and their cell counts);
  (b) steric / unbound genome ratio at k = 8;
  (c) fraction misclassified DETERMINISTIC at k relative to the k = 32 run.  Prefix
      classes are monotone (a genome DET at k is DET at every k' < k), so the
      misclassified set at k is DET(k) minus DET(32) and its size is a tally difference.
The reference semantics (not the paper's prose) are the target: SURVEY.md section 0
records the reference's own values (71 mixed hashes, ratio 0.124, 106 DET hashes).

usage: python tools/acceptance_s28.py [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2205_15311_b200.classify import enumerate_space  # noqa: E402
from paper_2205_15311_b200.genome import SearchSpace  # noqa: E402

KS = (1, 2, 4, 8, 16, 32)


def run() -> dict:
    t0 = time.time()
    h = enumerate_space(SearchSpace(2, 8), d=19, ks=KS, hist_k=8, seed=0, batch_size=1 << 24)
    el = time.time() - t0
    tal = h.tallies  # [q, 5]: DET, TRIV, STERIC, UNB, ERROR
    n = int(tal[0].sum())
    mixed = np.nonzero((h.det > 0) & (h.steric > 0))[0]
    det32 = int(tal[KS.index(32), 0])
    mis = {str(k): (int(tal[i, 0]) - det32) / n for i, k in enumerate(KS)}
    k8 = KS.index(8)
    return {
        "space": "S_(2,8)", "genomes": n, "d": 19, "seed": 0, "strict": True, "ks": list(KS), "hist_k": 8,
        "tallies": {str(k): dict(zip(("det", "trivial", "steric", "unbound", "error"), map(int, tal[i])))
                    for i, k in enumerate(KS)},
        "a_mixed_hashes": int(mixed.size),
        "a_mixed_cells": sorted(int(c) for c in h.cells[mixed]),
        "det_hashes": int(np.count_nonzero(h.det)),
        "b_steric_over_unbound_k8": int(tal[k8, 2]) / max(1, int(tal[k8, 3])),
        "c_misclassified_det_vs_k32": mis,
        "c_non_increasing": all(mis[str(a)] >= mis[str(b)] for a, b in zip(KS, KS[1:])),
        "seconds": el,
    }


if __name__ == "__main__":
    res = run()
    txt = json.dumps(res, indent=1)
    print(txt)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(txt + "\n")
