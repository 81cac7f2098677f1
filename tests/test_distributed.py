"""Multi-rank histogram exchange over gloo (world size 2, CPU): the same
allreduce_histogram code the NCCL path runs.  Each rank aggregates the
reference's golden per-genome rows of ITS round-robin chunks; the exchanged
result must equal the histogram of the whole slice on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests import _golden as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _hist_of(c, rows):
    from paper_2205_15311_b200.classify import Histogram
    e = c["expected"]
    return Histogram.from_rows(c["idx"][rows], e["cls"][rows], e["hash"][rows], e["w"][rows], e["h"][rows],
                               e["cells"][rows], e["shape"][rows], c["ks"], c["hist_k"], W=5)


def _worker(rank, world, port, name, chunk, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2205_15311_b200.classify import chunk_plan
    from paper_2205_15311_b200.distributed import allreduce_histogram, rank_chunks
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        c = G.slice_case(name)
        n = c["idx"].shape[0]
        mine = rank_chunks(chunk_plan(0, n, chunk), rank, world)
        rows = np.concatenate([np.arange(s, s + k) for s, k in mine]) if mine else np.zeros(0, np.int64)
        local = _hist_of(c, rows)
        merged = allreduce_histogram(local, None)
        full = _hist_of(c, np.arange(n))
        ok = merged == full
        q.put((rank, ok, len(merged), merged.total))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,chunk", [("s28_800000", 256), ("s32_rand", 1000), ("s28_rand_k32", 100)])
def test_allreduce_histogram_gloo_world2(name, chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, chunk, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, nkeys, total in res:
        assert ok, (rank, nkeys, total)
    assert res[0][2:] == res[1][2:]


def test_rank_chunks_partition():
    from paper_2205_15311_b200.classify import chunk_plan
    from paper_2205_15311_b200.distributed import rank_chunks
    plan = chunk_plan(100, 1000, 64)
    for world in (1, 2, 3, 8):
        parts = [rank_chunks(plan, r, world) for r in range(world)]
        got = sorted(i for p in parts for s, k in p for i in range(s, s + k))
        assert got == list(range(100, 1100))


def test_histogram_merge_commutative_associative():
    from paper_2205_15311_b200.classify import Histogram
    c = G.slice_case("s28_rand")
    n = c["idx"].shape[0]
    parts = [_hist_of(c, np.arange(i, n, 3)) for i in range(3)]
    full = _hist_of(c, np.arange(n))
    assert Histogram.merge_many(parts) == full
    assert parts[0].merge(parts[1]).merge(parts[2]) == parts[2].merge(parts[0].merge(parts[1]))
