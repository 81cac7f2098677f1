"""torchrun worker for tests/test_gpu_multirank.py: distributed.sweep_distributed (GA replicas
dealt over the ranks, one all_gather_object) with several ranks sharing the test GPU over gloo.
Prints one JSON line per rank comparing the rows with the single-process evolve.sweep."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from paper_2205_15311_b200 import evolve as E
    from paper_2205_15311_b200.distributed import sweep_distributed
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    base = E.GAConfig(pop_size=512, cutoff=3000)
    grid, runs = [0.3, 4.0], 21
    rows = sweep_distributed(grid, runs, base, seed0=3, sample_size=50, resamples=400)
    ref = E.sweep(grid, runs, base, seed0=3, sample_size=50, resamples=400)
    print(json.dumps({"rank": rank, "equal": rows == ref, "rows": rows}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
