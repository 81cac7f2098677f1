"""Does the GA generation rate depend on what was allocated before its buffers (physical placement
across the two dies' L2)?  Development aid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2205_15311_b200 import evolve as E

def rate(tag):
    ga = E.DeviceGA(1 << 20, 32, 0.3, "asexual")
    ga.run(1, 0, 50, 25, 1 << 20, 0)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        ga.run(1, 50, 2000, 25, 1 << 20, 0)
        best = min(best, time.perf_counter() - t)
    ga.close()
    print(f"{tag}: {2000 / best:.0f} gens/s ({best / 2000 * 1e6:.2f} us/gen)", flush=True)

rate("fresh")
bufs = [torch.empty(256 << 20, dtype=torch.uint8, device="cuda")]
rate("after 256 MB")
bufs.append(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
rate("after +64 MB")
for i in range(6):
    bufs.append(torch.empty((8 + i) << 20, dtype=torch.uint8, device="cuda"))
    rate(f"after +{8 + i} MB")
