"""Paper-scale GA sweep timing (Figs. 9-10: N = 512, L = 32, cutoff 20000,
100 runs per muL): one replica launch per sweep point vs sequential single-run launches.

usage: python tools/sweep_bench.py [runs]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2205_15311_b200 import evolve as E  # noqa: E402


def main(runs: int = 100) -> dict:
    out = {"runs_per_point": runs, "points": []}
    E.run_replicas(E.GAConfig(cutoff=100, stop_when="never"), [0, 1])  # warm-up
    for mu in (0.03, 0.1, 0.3, 1.0, 4.0):
        cfg = E.GAConfig(mu_L=mu, stop_when="never")  # full 20000 generations: fixed work per run
        torch.cuda.synchronize()
        t = time.perf_counter()
        recs = E.run_replicas(cfg, range(runs))
        el = time.perf_counter() - t
        gens = sum(r.generations for r in recs)
        t = time.perf_counter()
        one = E.run_ga(cfg, seed=0)
        el1 = time.perf_counter() - t
        assert one.generations == recs[0].generations and (one.count_at_target == recs[0].count_at_target).all()
        out["points"].append({"muL": mu, "replica_seconds": el, "replica_generations_per_s": gens / el,
                              "single_run_seconds": el1, "single_run_generations_per_s": one.generations / el1,
                              "speedup_vs_sequential_runs": (el1 * runs) / el})
    return out


if __name__ == "__main__":
    print(json.dumps(main(int(sys.argv[1]) if len(sys.argv) > 1 else 100), indent=1))
