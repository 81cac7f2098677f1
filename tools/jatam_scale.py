"""JaTAM GA generation time vs population (is the fitness pass floor- or throughput-bound?),
with the fitness memo on or off (TV_FITMEMO).  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2205_15311_b200 import _lib, assembly as A, evolve as E
from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
S28 = SearchSpace(2, 8)
tgt_idx = 0x801772
target = A.assemble_once(decode_tileset(genome_at_index(S28, tgt_idx), S28), 19, seed=0, genome_index=tgt_idx,
                         run_index=0).grid.cells >= 0
for lg in (18, 20, 22):
    n = 1 << lg
    ga = E.DeviceGA(n, 24, 0.3, "asexual")
    ga.set_population(np.random.default_rng(11).integers(0, 1 << 24, n, dtype=np.uint64))
    st = torch.cuda.current_stream()
    sp = _lib.ctypes.c_void_p(st.cuda_stream)
    ga.run_jatam(S28, target, 5, 0, 2, 361, stream=sp)
    out = []
    for g0, gens in ((2, 10), (12, 10), (22, 20)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(st)
        ga.run_jatam(S28, target, 5, g0, gens, 361, stream=sp)
        e1.record(st); torch.cuda.synchronize()
        out.append(f"gens {g0}-{g0 + gens}: {e0.elapsed_time(e1) / gens:.3f} ms/gen")
    print(f"memo={os.environ.get('TV_FITMEMO', '1')} n=2^{lg}: " + ", ".join(out), flush=True)
    ga.close()
