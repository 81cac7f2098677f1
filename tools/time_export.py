"""Time the first export of a full S_{2,8} device histogram (includes the representative-payload
fix-up launch) against a second, fix-up-free export.  Development aid for the payload path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2205_15311_b200 import classify as C
from paper_2205_15311_b200.genome import SearchSpace
dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 16)
dh.enumerate_range(SearchSpace(2, 8), 0, 1 << 24, 19, 0, True)
torch.cuda.synchronize()
t0 = time.perf_counter(); h1 = dh.export(); t1 = time.perf_counter(); h2 = dh.export(); t2 = time.perf_counter()
assert h1 == h2
print(f"{os.environ.get('TV_LIB_PATH')} threads={os.environ.get('TV_FAST_THREADS')}: first export {1e3*(t1-t0):.2f} ms, "
      f"second {1e3*(t2-t1):.2f} ms, {len(h1)} records")
