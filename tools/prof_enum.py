"""Profiling driver: time the enumeration kernel in histogram mode and classify mode."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2205_15311_b200 import _lib, _kernels
from paper_2205_15311_b200.classify import DeviceHistogram
from paper_2205_15311_b200.genome import SearchSpace, space_from_preset

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--start", type=int, default=0)
ap.add_argument("--space", default="s28")
ap.add_argument("--mode", default="both")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
sp = SearchSpace(2, 8) if a.space == "s28" else space_from_preset("s32_3_8")
ks = (1, 2, 4, 8) if a.space == "s28" else (7,)
stream = torch.cuda.current_stream()
spp = _lib.ctypes.c_void_p(stream.cuda_stream)

def timed(f):
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); f(); e1.record(stream); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)

if a.mode in ("both", "hist"):
    h = DeviceHistogram(ks, ks[-1], 5, 1 << 16)
    def f():
        h.clear(spp); h.enumerate_range(sp, a.start, a.n, 19, 0, True, spp)
    ms = timed(f)
    print(f"hist mode  n={a.n}: {ms:.3f} ms  {a.n/ms/1e3:.1f} M genomes/s  {_lib.launch_info()}")
if a.mode in ("both", "classify"):
    n = a.n
    dev = [torch.zeros((n, len(ks)), dtype=torch.uint8, device="cuda"), torch.zeros(n, dtype=torch.uint32, device="cuda"),
           torch.zeros(n, dtype=torch.uint8, device="cuda"), torch.zeros(n, dtype=torch.uint8, device="cuda"),
           torch.zeros(n, dtype=torch.uint16, device="cuda"), torch.zeros((n, 6), dtype=torch.uint64, device="cuda")]
    idx = (torch.arange(n, dtype=torch.int64, device="cuda") + a.start).view(torch.uint64)
    aa, bpl, mp, mv, fp = sp.kernel_args()
    def g():
        _kernels.classify_batch(idx, aa, bpl, mp, mv, fp, 19, np.array(ks), ks[-1], np.uint64(0), True, *dev)
    ms = timed(g)
    print(f"classify   n={a.n}: {ms:.3f} ms  {a.n/ms/1e3:.1f} M genomes/s  {_lib.launch_info()}")
