"""GA generation rate measured the way bench.py measures it (after an S_{2,8} enumeration and
its allocations in the same process), with the placement calibration logged
(TV_GA_CALIB_LOG=1).  Development aid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2205_15311_b200 import classify as C, evolve as E


def rate(tag):
    ga = E.DeviceGA(1 << 20, 32, 0.3, "asexual")
    ga.run(7, 0, 50, 25, 1 << 20, 0)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        ga.run(7, 50, 2000, 25, 1 << 20, 0)
        best = min(best, time.perf_counter() - t)
    ga.close()
    print(f"{tag}: {2000 / best:.0f} gens/s ({best / 2000 * 1e6:.2f} us/gen)", flush=True)


rate("fresh")
sp = C.PRESETS["s28_2_8"] if hasattr(C, "PRESETS") else None
bufs = [torch.empty(1 << 30, dtype=torch.uint8, device="cuda")]
rate("after 1 GiB torch")
bufs.append(torch.empty(300 << 20, dtype=torch.uint8, device="cuda"))
rate("after +300 MiB")
for i in range(4):
    bufs.append(torch.empty((37 + 13 * i) << 20, dtype=torch.uint8, device="cuda"))
    rate(f"after +{37 + 13 * i} MiB")
