"""Time one full S_{2,8} enumeration and one 2^24 block of S32 (best of 3, host clock around a
synchronised call); TV_LIB_PATH selects an alternate build for A/B runs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2205_15311_b200 import classify as C
from paper_2205_15311_b200.genome import SearchSpace, space_from_preset
dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 16)
d7 = C.DeviceHistogram((7,), 7, 5, 1 << 20)
def t(f):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3
a = t(lambda: (dh.clear(), dh.enumerate_range(SearchSpace(2, 8), 0, 1 << 24, 19, 0, True)))
S32 = space_from_preset("s32_3_8")
b = t(lambda: (d7.clear(), d7.enumerate_range(S32, 0x9E370000, 1 << 24, 19, 0, True)))
print(f"{os.environ.get('TV_LIB_PATH')} EU={os.environ.get('TV_EARLY_UNBOUND')}: S28 {a:.2f} ms  S32[16M] {b:.2f} ms  tallies {dh.export().tallies[3].tolist()} {d7.export().tallies[0].tolist()}")
