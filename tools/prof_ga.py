"""Time the device GA generation loop (Fujiyama, no early stop)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2205_15311_b200 import evolve as E

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--gens", type=int, default=2000)
ap.add_argument("--mode", default="asexual")
ap.add_argument("--mu", type=float, default=0.3)
a = ap.parse_args()
ga = E.DeviceGA(a.n, 32, a.mu, a.mode)
ga.run(1, 0, 50, 25, a.n, 0)
torch.cuda.synchronize()
t = time.perf_counter()
k, b, s, c = ga.run(1, 50, a.gens, 25, a.n, 0)
el = time.perf_counter() - t
print(f"GA n={a.n} mode={a.mode} mu={a.mu}: {k} gens in {el*1e3:.1f} ms -> {k/el:.0f} gens/s "
      f"({el/k*1e6:.2f} us/gen), mean fitness {s[-1]/a.n:.2f} best {b[-1]}")
