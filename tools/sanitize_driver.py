"""Small invocations of every device path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): classify_batch (pre-pass + sort + k_classify_fast, generic kernel),
histogram mode (k_prepass, k_classify_fast, k_hist_* merge / export / payload fix-up), the
device-row exchange (tv_hist_pack / replace_rows), canonical labels, the single-genome kernels,
the GA (k_ga_run, k_ga_replicas, JaTAM fitness and the fused JaTAM generations, wide genomes,
the mutation benchmark).  Sizes are small so racecheck finishes.

usage: compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2205_15311_b200 import _kernels, assembly as A, classify as C, evolve as E  # noqa: E402
from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index, space_from_preset  # noqa: E402

N = int(os.environ.get("SAN_N", 8192))


def outs(n, q, W=6):
    return [np.zeros((n, q), np.uint8), np.zeros(n, np.uint32), np.zeros(n, np.uint8), np.zeros(n, np.uint8),
            np.zeros(n, np.uint16), np.zeros((n, W), np.uint64)]


S28, S32 = SearchSpace(2, 8), space_from_preset("s32_3_8")
for sp, ks, hk in ((S28, (1, 2, 4, 8), 8), (S32, (7,), 7), (SearchSpace(4, 8), (2, 4), 4)):
    a, bpl, mp, mv, fp = sp.kernel_args()
    idx = np.random.default_rng(1).integers(0, sp.cardinality, N if sp.a <= 3 else 256, dtype=np.uint64)
    o = outs(idx.shape[0], len(ks))
    _kernels.classify_batch(idx, a, bpl, mp, mv, fp, 19, np.array(ks), hk, np.uint64(0), True, *o)
    print("classify_batch", sp.a, sp.b, "ok", flush=True)
h = C.enumerate_space(S28, ks=(1, 2, 4, 8), start=0x800000, count=N, batch_size=N // 2)
h32 = C.enumerate_space(S32, ks=(7,), start=0x9E370000, count=N, batch_size=N)
print("enumerate_space", len(h), len(h32), flush=True)
dh = C.DeviceHistogram((1, 2, 4, 8), 8, C.shape_words_for(19), 1 << 14)
dh.enumerate_range(S28, 0, N, 19, 0, True)
rows = np.zeros((1 << 14, dh.row_width), np.uint64)
tal = np.zeros((4, 5), np.int64)
n = dh.pack_into(rows, tal)
dh.replace_rows(np.ascontiguousarray(rows[:n]), tal)
dh.export()
dh.close()
print("pack/replace_rows", n, flush=True)
C.shape_labels(h.w, h.h, h.shape)
t = decode_tileset(genome_at_index(S28, 0x801772), S28)
A.classify_tileset(t, 19, 8, seed=0, genome_index=0x801772)
A.assemble_once(t, 19, seed=0, genome_index=0x801772)
print("single-genome ok", flush=True)
E.run_ga(E.GAConfig(pop_size=4096, length=32, mu_L=0.3, cutoff=20, stop_when="never"), seed=1)
E.run_ga(E.GAConfig(pop_size=2048, length=48, mu_L=1.0, mode="uniform", cutoff=10, stop_when="never"), seed=2)
E.run_replicas(E.GAConfig(pop_size=512, mu_L=0.3, cutoff=30, stop_when="never"), range(4))
E.run_ga(E.GAConfig(pop_size=3000, length=20, mu_L=0.5, cutoff=50, stop_when="discovery"), seed=3)  # staged stop
tgt = A.assemble_once(t, 19, seed=0, genome_index=0x801772).grid.cells >= 0
E.run_ga(E.GAConfig(pop_size=4096, length=24, mu_L=0.3, cutoff=3, stop_when="never",
                    init=np.random.default_rng(3).integers(0, 1 << 24, 4096, dtype=np.uint64)),
         fitness=E.JatamFitness(S28, tgt), seed=3)
ga = E.DeviceGA(4096, 24, 0.3, "asexual")  # fused JaTAM generations (pre-pass fitness cache, counting sort)
ga.set_population(np.random.default_rng(4).integers(0, 1 << 24, 4096, dtype=np.uint64))
ga.run_jatam(S28, tgt, 5, 0, 3, 300)
ga.close()
E.run_ga(E.GAConfig(pop_size=2048, length=100, mu_L=1.0, mode="single_point", cutoff=5, stop_when="never"), seed=6)
import torch  # noqa: E402
pop = torch.zeros(16 * 2048, dtype=torch.int64, device="cuda")
E.mutate_population(pop, 1024, 0.5, "distribution", count_flips=True)
E.mutate_population(pop, 1024, 0.5, "bitwise", count_flips=True)
print("GA ok", flush=True)
