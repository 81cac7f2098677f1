"""Per-pop latency of a lone lane: classify one long S_{2,8} genome (6247553: 8 UNBOUND runs, 1747 pops
in the reference; with TV_EARLY_UNBOUND=0 all 8 runs execute) in a launch of its own.  Development aid
(run under ncu for the kernel duration and stall reasons)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2205_15311_b200 import _kernels as K
from paper_2205_15311_b200.genome import SearchSpace
S28 = SearchSpace(2, 8)
a, bpl, mp, mv, fp = S28.kernel_args()
ks = np.array([1, 2, 4, 8], np.int64)
for idx in (6247553, 0x801772):
    ind = np.array([idx], np.uint64)
    outs = [np.zeros((1, 4), np.uint8), np.zeros(1, np.uint32), np.zeros(1, np.uint8), np.zeros(1, np.uint8),
            np.zeros(1, np.uint16), np.zeros((1, 6), np.uint64)]
    for rep in range(3):
        K.classify_batch(ind, a, bpl, mp, mv, fp, 19, ks, 8, 0, True, *outs)
    print(idx, outs[0].tolist(), flush=True)
