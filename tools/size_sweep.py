"""Device time of one S_{2,8} enumeration launch sequence (pre-pass, sort, classify) vs. the
number of genomes (CUDA events, best of 3): how the fixed and tail costs scale down for the
per-GPU shares of a multi-GPU run.  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2205_15311_b200 import classify as C
from paper_2205_15311_b200.genome import SearchSpace
dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 16)
sp = SearchSpace(2, 8)
s = torch.cuda.current_stream()
for lg in (18, 19, 20, 21, 22, 23, 24):
    n = 1 << lg
    best = 1e9
    for _ in range(3):
        dh.clear()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        if n >= 1 << 20:  # rank 0's share of a 2^24 / n-GPU run: 2^20 chunks round-robin
            dh.enumerate_chunks(sp, 0, n, 1 << 20, (1 << 20) * ((1 << 24) // n), 19, 0, True)
        else:
            dh.enumerate_range(sp, 0x5A0000, n, 19, 0, True)
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"2^{lg}: {best:.3f} ms  {n / best / 1e3:.0f} M genomes/s  (ideal from 2^24 rate: {n / (1 << 24) * 26.8:.3f} ms)")
