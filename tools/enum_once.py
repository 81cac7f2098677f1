"""One enumeration launch for profiling: full S_{2,8} (default) or a 2^24 block of S32.

usage: python tools/enum_once.py [s28|s32]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2205_15311_b200 import classify as C  # noqa: E402
from paper_2205_15311_b200.genome import SearchSpace, space_from_preset  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "s28"
if which == "s28":
    dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 16)
    dh.enumerate_range(SearchSpace(2, 8), 0, 1 << 24, 19, 0, True)
else:
    dh = C.DeviceHistogram((7,), 7, 5, 1 << 20)
    dh.enumerate_range(space_from_preset("s32_3_8"), 0x9E370000, 1 << 24, 19, 0, True)
torch.cuda.synchronize()
h = dh.export()
C.shape_labels(h.w, h.h, h.shape)  # one k_shape_labels launch over the records
torch.cuda.synchronize()
