"""Multi-rank histogram exchange over gloo (world sizes 2 and 4, CPU): the key-partitioned
exchange (owner = hash mod R, all_to_all, owner-side merge, all_gather of the disjoint
shards) that the NCCL path runs with a device-side merge.  Each rank aggregates the
reference's golden per-genome rows of ITS round-robin chunks; the exchanged result must
equal the histogram of the whole slice on every rank, and the owned shards must
partition it."""
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
    from paper_2205_15311_b200.distributed import allreduce_histogram, owner_of, rank_chunks
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        c = G.slice_case(name)
        n = c["idx"].shape[0]
        mine = rank_chunks(chunk_plan(0, n, chunk), rank, world)
        rows = np.concatenate([np.arange(s, s + k) for s, k in mine]) if mine else np.zeros(0, np.int64)
        local = _hist_of(c, rows)
        merged = allreduce_histogram(local, None)
        shard = allreduce_histogram(local, None, sharded=True)
        full = _hist_of(c, np.arange(n))
        ok = merged == full
        own = np.nonzero(owner_of(full.keys.astype(np.int64), world) == rank)[0]
        shard_ok = (np.array_equal(shard.keys, full.keys[own]) and np.array_equal(shard.shape, full.shape[own])
                    and np.array_equal(shard.rep_any, full.rep_any[own]) and np.array_equal(shard.det, full.det[own])
                    and np.array_equal(shard.tallies, full.tallies))
        q.put((rank, bool(ok) and bool(shard_ok), len(merged), merged.total, bool(ok), bool(shard_ok)))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("name,chunk,world", [("s28_800000", 256, 2), ("s32_rand", 1000, 2), ("s28_rand_k32", 100, 2),
                                              ("s28_800000", 300, 4), ("s28_rand", 20000, 4)])
def test_allreduce_histogram_gloo(name, chunk, world):
    """world 4 with 20000-index chunks of s28_rand: some ranks hold no genomes at all."""
    res = _spawn(_worker, world, name, chunk)
    for rank, ok, nkeys, total, *detail in res:
        assert ok, (rank, nkeys, total, detail)
    assert len({r[2:4] for r in res}) == 1


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


def _collision_rows():
    """Synthetic per-genome rows: hash 0xABC carried by two different shapes (a 32-bit
    collision), genome 7 (lowest index) holds shape A, genomes 9 and 12 shape B."""
    idx = np.array([12, 9, 7, 3], np.uint64)
    cls = np.array([[0], [2], [0], [1]], np.uint8)
    hsh = np.array([0xABC, 0xABC, 0xABC, 0], np.uint32)
    w = np.array([2, 2, 1, 0], np.uint8)
    h = np.array([1, 1, 3, 0], np.uint8)
    cells = np.array([2, 2, 3, 0], np.uint16)
    shape = np.zeros((4, 5), np.uint64)
    shape[[0, 1], 0] = 3
    shape[2, 0] = 7
    return idx, cls, hsh, w, h, cells, shape


def test_payload_is_the_representatives():
    """Payload (w, h, cells, bitmap) of a key = that of its lowest-index genome, whatever
    the row order or merge order (the device histogram follows the same rule)."""
    from paper_2205_15311_b200.classify import Histogram
    idx, cls, hsh, w, h, cells, shape = _collision_rows()
    for perm in ([0, 1, 2, 3], [2, 3, 1, 0], [3, 0, 2, 1]):
        H = Histogram.from_rows(idx[perm], cls[perm], hsh[perm], w[perm], h[perm], cells[perm], shape[perm], (1,), 1)
        assert H.keys.tolist() == [0xABC] and int(H.rep_any[0]) == 7
        assert (int(H.w[0]), int(H.h[0]), int(H.cells[0]), int(H.shape[0, 0])) == (1, 3, 3, 7)
    a = Histogram.from_rows(idx[:2], cls[:2], hsh[:2], w[:2], h[:2], cells[:2], shape[:2], (1,), 1)
    b = Histogram.from_rows(idx[2:], cls[2:], hsh[2:], w[2:], h[2:], cells[2:], shape[2:], (1,), 1)
    for m in (Histogram.merge_many([a, b]), Histogram.merge_many([b, a])):
        assert (int(m.w[0]), int(m.cells[0]), int(m.shape[0, 0]), int(m.det[0]), int(m.steric[0])) == (1, 3, 7, 2, 1)


def _collision_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2205_15311_b200.classify import Histogram
    from paper_2205_15311_b200.distributed import allreduce_histogram
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        idx, cls, hsh, w, h, cells, shape = _collision_rows()
        rows = [0, 1] if rank == 0 else [2, 3]  # rank 1 holds the representative (genome 7)
        local = Histogram.from_rows(idx[rows], cls[rows], hsh[rows], w[rows], h[rows], cells[rows], shape[rows],
                                    (1,), 1, W=5)
        m = allreduce_histogram(local, None)
        q.put((rank, int(m.rep_any[0]), int(m.w[0]), int(m.h[0]), int(m.cells[0]), int(m.shape[0, 0])))
    finally:
        dist.destroy_process_group()


def test_allreduce_payload_from_representative_rank():
    res = _spawn(_collision_worker, 2)
    for r in res:
        assert r[1:] == (7, 1, 3, 3, 7), r


# ---------------------------------------------------------------- GA sweeps over ranks (replicas only)
class _FakeRun:
    def __init__(self, discovery, adaptation):
        self.discovery, self.adaptation = discovery, adaptation


def _fake_runner(cfg, seeds):
    """Deterministic stand-in for evolve.sweep_runs (no GPU here): per-run times as a function
    of (muL, seed), censored (None) often enough to exercise both SPEC:448 branches."""
    out = []
    for s in seeds:
        r = np.random.default_rng(int(s) * 7919 + int(round(cfg.mu_L * 1000)))
        p = 0.2 if cfg.mu_L < 1 else 0.7
        d = None if r.random() < p else int(r.integers(1, cfg.cutoff))
        a = None if (d is None or r.random() < p) else int(r.integers(d, cfg.cutoff))
        out.append(_FakeRun(d, a))
    return out


def _sweep_worker(rank, world, port, out_dir, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2205_15311_b200 import evolve as E
    from paper_2205_15311_b200.distributed import sweep_distributed
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        grid, runs = [0.1, 0.3, 4.0], 37
        base = E.GAConfig(cutoff=500)
        out = os.path.join(out_dir, "sweep.json")
        rows = sweep_distributed(grid, runs, base, seed0=11, sample_size=40, resamples=500, out=out,
                                 runner=_fake_runner)
        ref = E.sweep(grid, runs, base, seed0=11, sample_size=40, resamples=500, runner=_fake_runner)
        dist.barrier()
        q.put((rank, rows == ref, os.path.exists(out), [r["adaptation"]["median"] is None for r in rows]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sweep_distributed_equals_sweep(world, tmp_path):
    """Run r of every point on rank r mod R, one all_gather_object: the rows equal the
    single-process sweep exactly (same seeds, same bootstrap), on every rank."""
    res = _spawn(_sweep_worker, world, str(tmp_path))
    assert sorted(r[0] for r in res) == list(range(world))
    assert all(r[1] for r in res), res
    assert all(r[2] for r in res)  # rank 0 wrote the sweep JSON
    assert res[0][3][-1] is True and res[0][3][0] is False  # both censoring branches occur
