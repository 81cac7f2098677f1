"""Time the JaTAM-shape-fitness GA generation (bench.py ga_jatam workload) and print the device
time of its launches vs the host-clock generation time (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_15311_b200 import assembly as A, evolve as E  # noqa: E402
from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index  # noqa: E402

S28 = SearchSpace(2, 8)
n = 1 << 20
tgt_idx = 0x801772
target = A.assemble_once(decode_tileset(genome_at_index(S28, tgt_idx), S28), 19, seed=0, genome_index=tgt_idx,
                         run_index=0).grid.cells >= 0
ga = E.DeviceGA(n, 24, 0.3, "asexual")
ga.set_population(np.random.default_rng(11).integers(0, 1 << 24, n, dtype=np.uint64))
st = torch.cuda.current_stream()
for g in range(3):
    f = ga.jatam_fitness(S28, target, 19, 8)
    ga.run(5, g, 1, 361, n, 0, f_ext=f)
torch.cuda.synchronize()
for rep in range(2):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t0 = time.perf_counter()
    e[0].record(st)
    f = ga.jatam_fitness(S28, target, 19, 8)
    e[1].record(st)
    ga.run(5, 3 + rep, 1, 361, n, 0, f_ext=f)
    e[2].record(st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"generation: host {1e3 * (t1 - t0):.3f} ms, fitness events {e[0].elapsed_time(e[1]):.3f} ms, "
          f"GA events {e[1].elapsed_time(e[2]):.3f} ms")
