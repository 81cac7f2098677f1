"""SPEC ACCEPTANCE 3 (hash integrity) on the device: do distinct DETERMINISTIC shape bitmaps
share a 32-bit shape hash?  Classifies every genome of the space with classify_batch on
device tensors (batches of 2^22), keeps the DET rows at k = ks[-1] and counts distinct
(hash, w, h, bitmap) payloads against distinct hashes.

usage: python tools/hash_integrity.py s28|s32 [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_15311_b200 import _kernels as K  # noqa: E402
from paper_2205_15311_b200.classify import collision_probability  # noqa: E402
from paper_2205_15311_b200.genome import SearchSpace, space_from_preset  # noqa: E402


def run(which: str, batch: int = 1 << 22) -> dict:
    sp, ks = (SearchSpace(2, 8), (8,)) if which == "s28" else (space_from_preset("s32_3_8"), (7,))
    a, bpl, mp, mv, fp = sp.kernel_args()
    n_all = sp.cardinality
    dev = "cuda"
    cls = torch.empty((batch, 1), dtype=torch.uint8, device=dev)
    hsh = torch.empty(batch, dtype=torch.uint32, device=dev)
    w = torch.empty(batch, dtype=torch.uint8, device=dev)
    h = torch.empty(batch, dtype=torch.uint8, device=dev)
    cells = torch.empty(batch, dtype=torch.uint16, device=dev)
    shape = torch.empty((batch, 5), dtype=torch.uint64, device=dev)
    acc = torch.zeros((0, 7), dtype=torch.int64, device=dev)
    t0 = time.time()
    for start in range(0, n_all, batch):
        idx = torch.arange(start, start + batch, dtype=torch.int64, device=dev).view(torch.uint64)
        K.classify_batch(idx, a, bpl, mp, mv, fp, 19, np.array(ks), ks[-1], np.uint64(0), True,
                         cls, hsh, w, h, cells, shape)
        det = cls[:, 0] == 0
        hs = hsh.view(torch.int32).to(torch.int64) & 0xFFFFFFFF  # (torch cannot index unsigned 32/64)
        rows = torch.cat([hs[det].view(-1, 1), (w[det].to(torch.int64) | (h[det].to(torch.int64) << 8)).view(-1, 1),
                          shape.view(torch.int64)[det]], dim=1)
        acc = torch.unique(torch.cat([acc, rows]), dim=0)  # distinct (hash, w|h<<8, bitmap) rows
    torch.cuda.synchronize()
    el = time.time() - t0
    npay = int(acc.shape[0])
    nhash = int(torch.unique(acc[:, 0]).numel())
    return {"space": which, "genomes": n_all, "k": ks[-1], "det_payloads": npay, "det_hashes": nhash,
            "colliding_hashes": npay - nhash,
            "birthday_expectation": npay * (npay - 1) / 2 / 2 ** 32,
            "collision_probability_1000": collision_probability(1000), "seconds": el}


if __name__ == "__main__":
    r = run(sys.argv[1] if len(sys.argv) > 1 else "s28")
    txt = json.dumps(r, indent=1)
    print(txt)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(txt + "\n")
