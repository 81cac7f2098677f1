"""Device time of the JaTAM-fitness pass vs population size (fresh random populations, no
fitness cache): where the fitness kernel's floor lies.  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2205_15311_b200 import assembly as A, evolve as E
from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
S28 = SearchSpace(2, 8)
tgt = 0x801772
target = A.assemble_once(decode_tileset(genome_at_index(S28, tgt), S28), 19, seed=0, genome_index=tgt,
                         run_index=0).grid.cells >= 0
st = torch.cuda.current_stream()
for lg in (14, 16, 18, 19, 20, 21, 22):
    n = 1 << lg
    ga = E.DeviceGA(n, 24, 0.3, "asexual")
    ga.set_population(np.random.default_rng(lg).integers(0, 1 << 24, n, dtype=np.uint64))
    ga.jatam_fitness(S28, target, 19, 8)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ga.jatam_fitness(S28, target, 19, 8)
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"2^{lg}: {best:.3f} ms  ({n / best / 1e3:.0f} M genomes/s)", flush=True)
    ga.close()
