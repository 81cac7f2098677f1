"""Save the bench ga_jatam population at a few generations (development aid: chain analysis)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2205_15311_b200 import assembly as A, evolve as E
from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
S28 = SearchSpace(2, 8)
n = 1 << 20
tgt_idx = 0x801772
target = A.assemble_once(decode_tileset(genome_at_index(S28, tgt_idx), S28), 19, seed=0, genome_index=tgt_idx,
                         run_index=0).grid.cells >= 0
ga = E.DeviceGA(n, 24, 0.3, "asexual")
ga.set_population(np.random.default_rng(11).integers(0, 1 << 24, n, dtype=np.uint64))
for g in range(21):
    f = ga.jatam_fitness(S28, target, 19, 8)
    if g in (2, 12, 20):
        np.save(f"gpurun_out/jatam_pop_g{g}.npy", ga.population())
        np.save(f"gpurun_out/jatam_fit_g{g}.npy", f.cpu().numpy().view(np.uint32))
    ga.run(5, g, 1, 361, n, 0, f_ext=f)
print("ok")
