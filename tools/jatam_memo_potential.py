"""How much of the JaTAM fitness work would a genome -> fitness memo table (across generations)
remove beyond the parent cache?  Runs the bench.py ga_jatam workload generation by generation
and counts, per generation, the children that are unmutated copies (parent cache), the other
children whose genome was already evaluated in an earlier generation or earlier in the same
population (memo), and the rest.  Development aid."""
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
pop = np.random.default_rng(11).integers(0, 1 << 24, n, dtype=np.uint64)
ga.set_population(pop)
seen = set()
gens = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for g in range(gens):
    f = ga.jatam_fitness(S28, target, 19, 8)
    fk = ga._h and None
    ga.run(5, g, 1, 361, n, 0, f_ext=f)
    child = ga.population()
    uniq, inv, cnt = np.unique(child, return_inverse=True, return_counts=True)
    prev = set(pop.tolist())
    # unmutated copies: equal to some genome of the parent population (upper bound of the parent cache)
    in_prev = np.isin(child, pop)
    in_seen = np.array([int(x) in seen for x in uniq.tolist()])[inv]
    distinct_new = np.unique(child[~in_prev & ~in_seen]).size
    seen.update(pop.tolist())
    print(f"gen {g:3d}: copies-of-a-parent-genome {in_prev.mean():.3f}  other, seen before {(~in_prev & in_seen).mean():.3f}  "
          f"other, new {(~in_prev & ~in_seen).mean():.3f} ({distinct_new} distinct)  distinct in population {uniq.size}  "
          f"best {int(f.cpu().numpy().view(np.uint32).max())}", flush=True)
    pop = child
