"""Projected 1/2/4/8-GPU strong scaling of the S_{2,8} and S^{32}_{3,8} benches, measured on ONE GPU.

For R ranks, every rank's share (chunk c -> rank c mod R) is enumerated into its own device
histogram, one after the other; the step time of R GPUs is projected as the slowest share's
enumeration time plus the measured cost of the exchange work one rank does (tv_hist_pack of
its rows, tv_hist_replace_rows of all R ranks' rows, export).  NVLink all_gather/all_reduce
time is not included (KB-MB payloads; NCCL latency ~10-50 us).  This is a projection, not a
multi-GPU measurement.

usage: python tools/scaling_projection.py [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2205_15311_b200 import _lib  # noqa: E402
from paper_2205_15311_b200.classify import DeviceHistogram  # noqa: E402
from paper_2205_15311_b200.genome import SearchSpace, space_from_preset  # noqa: E402


def share_time(dh, sp, ks, rank, world, chunk, n_all):
    a, bpl, mp, mv, fp = sp.kernel_args()
    L = _lib.lib()
    import numpy as np
    k = np.array(ks, np.int64)
    mine = len(range(rank, n_all // chunk, world))
    dh.clear()
    torch.cuda.synchronize()
    t = time.perf_counter()
    _lib.check(L.tv_enumerate_chunks(rank * chunk, mine * chunk, chunk, chunk * world, a, bpl, _lib.ptr(mp),
                                     _lib.ptr(mv), mp.shape[0], _lib.ptr(fp), fp.shape[0], 19, _lib.ptr(k), k.shape[0],
                                     ks[-1], 0, 1, dh._h, None))
    torch.cuda.synchronize()
    return time.perf_counter() - t


def project(name, sp, ks, n_all, chunk, worlds=(1, 2, 4, 8), cap=1 << 21):
    rows = []
    base = None
    w = DeviceHistogram(ks, ks[-1], 5, cap)  # warm the allocator pool with the largest share (R = 1)
    share_time(w, sp, ks, 0, 1, chunk, n_all)
    w.close()
    for R in (worlds[-1],) + tuple(worlds):  # the first pass warms up allocations and kernels
        warm = base is None and not rows and R == worlds[-1] and len(rows) == 0 and not hasattr(project, "_w" + name)
        hs = [DeviceHistogram(ks, ks[-1], 5, cap) for _ in range(R)]
        ts = [share_time(hs[r], sp, ks, r, R, chunk, n_all) for r in range(R)]
        if R == 1:
            t0 = time.perf_counter()
            hs[0].export()
            ex = time.perf_counter() - t0
        else:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            packs = []
            tal = torch.zeros((len(ks), 5), dtype=torch.int64, device="cuda")
            for r in range(R):
                n = hs[r].count()[0]
                rr = torch.zeros((max(n, 1), hs[r].row_width), dtype=torch.int64, device="cuda")
                t = torch.zeros((len(ks), 5), dtype=torch.int64, device="cuda")
                hs[r].pack_into(rr, t)
                packs.append(rr)
                tal += t
            pack_t = (time.perf_counter() - t0) / R  # one rank packs its own rows
            t1 = time.perf_counter()
            hs[0].replace_rows(torch.cat(packs), tal)
            hs[0].export()
            ex = pack_t + time.perf_counter() - t1
        step = max(ts) + ex
        if warm:
            setattr(project, "_w" + name, True)
            for h in hs:
                h.close()
            continue
        if base is None:
            base = step
        rows.append({"gpus": R, "slowest_share_ms": max(ts) * 1e3, "exchange_ms": ex * 1e3, "step_ms": step * 1e3,
                     "genomes_per_s": n_all / step, "efficiency": base / (R * step)})
        for h in hs:
            h.close()
    return {"workload": name, "rows": rows}


if __name__ == "__main__":
    out = {"note": __doc__.split("\n\n")[1].replace("\n", " "),
           "s28": project("full S_(2,8), ks=(1,2,4,8), 2^20-index chunks", SearchSpace(2, 8), (1, 2, 4, 8), 1 << 24,
                          1 << 20, cap=1 << 16),
           "s32": project("full S^32_(3,8), k=7, 2^24-index chunks", space_from_preset("s32_3_8"), (7,), 1 << 32,
                          1 << 24, worlds=(1, 8))}
    txt = json.dumps(out, indent=1)
    print(txt)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(txt + "\n")
