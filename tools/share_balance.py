"""Per-rank share time of the S_{2,8} bench at N ranks (each share enumerated alone on this GPU,
CUDA events, best of 2) for two round-robin chunk sizes: how even the shares are.  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2205_15311_b200 import classify as C
from paper_2205_15311_b200.genome import SearchSpace
dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 16)
sp = SearchSpace(2, 8)
s = torch.cuda.current_stream()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for lg in (20, 18, 16):
    chunk = 1 << lg
    ts = []
    for r in range(N):
        best = 1e9
        for _ in range(2):
            dh.clear()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            dh.enumerate_chunks(sp, r * chunk, (1 << 24) // N, chunk, chunk * N, 19, 0, True)
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        ts.append(best)
    print(f"N={N} chunk=2^{lg}: max {max(ts):.2f} ms, mean {sum(ts)/N:.2f}, min {min(ts):.2f}  "
          f"-> {(1 << 24) / max(ts) / 1e3:.0f} M genomes/s aggregate")
