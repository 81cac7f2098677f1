"""Fitness-pass time (k_prepass + sort + k_classify_fast fit mode, no caches) vs the number of
genomes, on an evolved JaTAM population (_scratch/jatam_pop_g12.npy from tools/jatam_dump_pop.py)
and on uniform S_{2,8} genomes.  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TV_FITCACHE"] = "0"
os.environ["TV_FITMEMO"] = "0"
import numpy as np, torch
from paper_2205_15311_b200 import assembly as A, evolve as E
from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
S28 = SearchSpace(2, 8)
tgt_idx = 0x801772
target = A.assemble_once(decode_tileset(genome_at_index(S28, tgt_idx), S28), 19, seed=0, genome_index=tgt_idx,
                         run_index=0).grid.cells >= 0
evolved = np.load("_scratch/jatam_pop_g12.npy")
rng = np.random.default_rng(1)
for name, src in (("evolved", evolved), ("uniform", rng.integers(0, 1 << 24, 1 << 20, dtype=np.uint64))):
    for lg in (14, 16, 17, 18, 19, 20):
        n = 1 << lg
        ga = E.DeviceGA(n, 24, 0.3, "asexual")
        ga.set_population(np.ascontiguousarray(src[rng.permutation(src.size)[:n]]))
        ga.jatam_fitness(S28, target, 19, 8)
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            ga.jatam_fitness(S28, target, 19, 8)
            e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{name} n=2^{lg}: {best:.3f} ms  ({n / best / 1e3:.0f} M genomes/s)", flush=True)
        ga.close()
