"""Does the enumeration time depend on where the launch's buffers land (like the GA loop,
DESIGN.md section 6)?  Times full S_{2,8} and a 2^24 S32 block after different earlier
allocations in one process.  Development aid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2205_15311_b200 import classify as C
from paper_2205_15311_b200.genome import SearchSpace, space_from_preset

S32 = space_from_preset("s32_3_8")


def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def rate(tag):
    dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 16)
    d7 = C.DeviceHistogram((7,), 7, 5, 1 << 20)
    a = t(lambda: (dh.clear(), dh.enumerate_range(SearchSpace(2, 8), 0, 1 << 24, 19, 0, True)))
    b = t(lambda: (d7.clear(), d7.enumerate_range(S32, 0x9E370000, 1 << 24, 19, 0, True)))
    print(f"{tag}: S28 {a:.2f} ms  S32[16M] {b:.2f} ms", flush=True)
    del dh, d7


rate("fresh")
bufs = []
for i, mb in enumerate((1024, 300, 37, 50, 63, 76, 89)):
    bufs.append(torch.empty(mb << 20, dtype=torch.uint8, device="cuda"))
    rate(f"after +{mb} MiB")
