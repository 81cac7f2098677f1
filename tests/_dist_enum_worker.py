"""torchrun worker for tests/test_gpu_multirank.py: enumerate_space_distributed with the
device-side exchange (key-partitioned all_to_all + tv_hist_replace_rows merge + payload
fix-up on the owner) over gloo, several ranks sharing the test GPU.  Prints one JSON line
per rank comparing the merged histogram with the single-GPU enumerate_space."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from paper_2205_15311_b200.classify import enumerate_space
    from paper_2205_15311_b200.distributed import enumerate_space_distributed
    from paper_2205_15311_b200.genome import SearchSpace, space_from_preset
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    res = {"rank": rank}
    cases = {"s28_idle": (SearchSpace(2, 8), (1, 2, 4, 8), 0x800000, 3000, 4096),   # one chunk: other ranks idle
             "s28_ragged": (SearchSpace(2, 8), (1, 2, 4, 8), 0x123456, 200_003, 1 << 14),
             "s32_block": (space_from_preset("s32_3_8"), (7,), 0x9E370000, 1 << 20, 1 << 16)}
    for name, (sp, ks, start, count, bs) in cases.items():
        got = enumerate_space_distributed(sp, ks=ks, start=start, count=count, batch_size=bs, device_exchange=True)
        ref = enumerate_space(sp, ks=ks, start=start, count=count, batch_size=1 << 20)
        res[name] = bool(got == ref)
        res[name + "_keys"] = len(got)
    print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
