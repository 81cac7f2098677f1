"""Multi-GPU enumeration: index-range sharding plus one key-partitioned histogram exchange.

Enumeration shards naturally -- every genome's substream is keyed by
(seed, enumeration index, run) (_k:45-48), so which rank processes an index
cannot change its result.  Chunks are dealt round-robin (chunk c -> rank
c mod R) because work varies strongly with the high index bits (the seed
tile's labels).  The only exchange is at the end, and it is O(keys) per rank:

1. every rank cuts its records by owner = shape hash mod R and sends each
   owner its part with one ``all_to_all`` (plus one all-reduce of the class
   tallies);
2. every owner merges what it received -- counts added, representatives
   lowered, payload = the representative's, so colliding shapes under one hash
   resolve exactly as the per-genome aggregation does;
3. the merged shards are disjoint by construction; ``gather_sharded`` concatenates
   them (one ``all_gather``) when a rank needs the whole table.

A rank therefore merges ~1/R of the rows instead of all R ranks' rows (the
round-1 all-gather-everything scheme).  With the NCCL backend the rows live in
HBM, the collectives run over NVLink and the merge is the device histogram's
(``tv_hist_replace_rows``); the host path (``allreduce_histogram``) runs the same
partition / all_to_all / merge / gather on gloo for the multi-process CPU tests.
"""
from __future__ import annotations

import numpy as np

from .classify import DeviceHistogram, Histogram, _space_meta, chunk_plan, shape_words_for  # noqa: F401

U64_MAX = np.iinfo(np.uint64).max


def _dev(group):
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def owner_of(keys, world: int):
    """Owning rank of each 32-bit shape hash (numpy or torch integer array)."""
    return (keys & 0xFFFFFFFF) % world


def _exchange(rows, owner, world: int, group, dev):
    """Send rows[i] to rank owner[i] (torch int64 [n, R] on ``dev``); returns the rows
    this rank received, grouped by source rank (one all_to_all for the counts, one
    for the rows)."""
    import torch
    import torch.distributed as dist
    order = torch.argsort(owner, stable=True)
    rows = rows[order].contiguous()
    send = torch.bincount(owner, minlength=world).to(torch.int64)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    sc, rc = send.tolist(), recv.tolist()
    out = torch.empty((sum(rc), rows.shape[1]), dtype=torch.int64, device=dev)
    dist.all_to_all_single(out, rows, output_split_sizes=rc, input_split_sizes=sc, group=group)
    return out, rc


# ---------------------------------------------------------------- host records <-> rows
def records_to_rows(h: Histogram) -> np.ndarray:
    """Histogram records as int64 rows {key, det, steric, rep_det, rep_any, whc, shape[W]}."""
    n = len(h)
    r = np.zeros((n, 6 + h.W), np.uint64)
    r[:, 0] = h.keys
    r[:, 1] = h.det
    r[:, 2] = h.steric
    r[:, 3] = h.rep_det
    r[:, 4] = h.rep_any
    r[:, 5] = (h.w.astype(np.uint64) | (h.h.astype(np.uint64) << np.uint64(8))
               | (h.cells.astype(np.uint64) << np.uint64(16)))
    r[:, 6:] = h.shape
    return r.view(np.int64)


def rows_to_records(rows: np.ndarray, like: Histogram, tallies=None) -> Histogram:
    """Inverse of records_to_rows (rows need not be sorted; keys must be unique)."""
    r = np.ascontiguousarray(rows).view(np.uint64)
    r = r[np.argsort(r[:, 0], kind="stable")]
    out = Histogram(like.ks, like.hist_k, like.W, meta=dict(like.meta))
    out.keys = r[:, 0].astype(np.uint32)
    out.det, out.steric, out.rep_det, out.rep_any = (r[:, i].copy() for i in (1, 2, 3, 4))
    out.w = (r[:, 5] & np.uint64(0xFF)).astype(np.uint8)
    out.h = ((r[:, 5] >> np.uint64(8)) & np.uint64(0xFF)).astype(np.uint8)
    out.cells = ((r[:, 5] >> np.uint64(16)) & np.uint64(0xFFFF)).astype(np.uint16)
    out.shape = np.ascontiguousarray(r[:, 6:]).reshape(r.shape[0], like.W)
    out.tallies = np.array(like.tallies if tallies is None else tallies, np.int64).reshape(like.tallies.shape)
    return out


def gather_sharded(part: Histogram, group=None) -> Histogram:
    """Concatenate key-disjoint shards (one per rank; tallies already global) into the
    whole histogram on every rank: one all_gather of the padded record rows."""
    import torch
    import torch.distributed as dist
    dev = _dev(group)
    world = dist.get_world_size(group)
    rows = torch.from_numpy(records_to_rows(part)).to(dev)
    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=dev)
    ns = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(ns, n, group=group)
    ns = ns.tolist()
    nmax = max(1, max(ns))
    pad = torch.zeros((nmax, rows.shape[1]), dtype=torch.int64, device=dev)
    pad[: rows.shape[0]] = rows
    allr = torch.empty((world * nmax, rows.shape[1]), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allr, pad, group=group)
    allr = allr.cpu().numpy().reshape(world, nmax, -1)
    return rows_to_records(np.concatenate([allr[r, : ns[r]] for r in range(world)]), part)


def allreduce_histogram(h: Histogram, group=None, sharded: bool = False) -> Histogram:
    """Combine per-rank host histograms by key ownership; every rank returns the identical
    merged result (or, with ``sharded``, the records it owns plus the global tallies)."""
    import torch
    import torch.distributed as dist
    dev = _dev(group)
    world = dist.get_world_size(group)
    rows = torch.from_numpy(records_to_rows(h)).to(dev)
    got, rc = _exchange(rows, owner_of(rows[:, 0], world), world, group, dev)
    tal = torch.from_numpy(np.array(h.tallies, np.int64)).to(dev)  # a copy: all_reduce works in place
    dist.all_reduce(tal, op=dist.ReduceOp.SUM, group=group)
    got = got.cpu().numpy()
    tal = tal.cpu().numpy()
    # one part per source rank (keys unique within a part), merged in rank order
    offs = np.r_[0, np.cumsum(rc)]
    parts = [rows_to_records(got[offs[r]:offs[r + 1]], h, np.zeros_like(tal)) for r in range(world)]
    mine = Histogram.merge_many(parts)
    mine.tallies = tal.reshape(h.tallies.shape).astype(np.int64)
    return mine if sharded else gather_sharded(mine, group)


def allreduce_device_histogram(dev: DeviceHistogram, group=None, meta: dict | None = None,
                               export: bool = True, stream=None) -> Histogram | None:
    """Device-resident, key-partitioned exchange (NCCL): each rank packs its raw records on
    the GPU (tv_hist_pack), cuts them by owner, one all_to_all moves each part to its owner
    over NVLink and one all_reduce sums the tallies; each owner merges its rows into its
    own device histogram (tv_hist_replace_rows: counts added, representatives lowered,
    payload = lowest owner).  ``dev`` then holds this rank's key shard of the merged
    histogram with the global tallies.  export=True exports the shard (the payload
    fix-up re-derives payloads whose owner is not the representative, each rank for its
    own keys) and gathers the whole table on every rank (same result as
    allreduce_histogram); export=False stops with the shard resident (returns None).
    Every call goes to ``stream`` (default: torch's current stream)."""
    import torch
    import torch.distributed as dist
    from . import _lib
    world = dist.get_world_size(group)
    st = stream if stream is not None else torch.cuda.current_stream()
    sp = _lib.ctypes.c_void_p(st.cuda_stream)
    dv = torch.device("cuda", torch.cuda.current_device())
    # collectives on the device for NCCL; other backends (gloo: several ranks sharing one GPU
    # in tests) move the same tensors through host memory
    cv = dv if dist.get_backend(group) == "nccl" else torch.device("cpu")
    with torch.cuda.stream(st):
        n_local, _ = dev.count(sp)
        rows = torch.zeros((max(1, n_local), dev.row_width), dtype=torch.int64, device=dv)
        tallies = torch.zeros((len(dev.ks), 5), dtype=torch.int64, device=dv)
        dev.pack_into(rows, tallies, sp)
        rows = rows[:n_local].to(cv)
        got, _ = _exchange(rows, owner_of(rows[:, 0], world), world, group, cv)
        tallies = tallies.to(cv)
        dist.all_reduce(tallies, op=dist.ReduceOp.SUM, group=group)
        dev.replace_rows(got.to(dv), tallies.to(dv), sp)
        if not export:
            return None
        part = dev.export(sp, meta=meta)
    return gather_sharded(part, group)


def sweep_distributed(mu_L_grid, runs: int = 100, base=None, seed0: int = 0, sample_size: int = 100,
                      resamples: int = 10000, out: str | None = None, group=None, runner=None) -> list[dict]:
    """evolve.sweep over all ranks of ``group`` (GA: replicas only).  Run r of
    every sweep point goes to rank r mod R, each rank launches its runs of a point at once
    (evolve.sweep_runs: one replica launch), and one all_gather_object brings every run's
    discovery / adaptation time to every rank.  Run r uses seed seed0 + r wherever it runs,
    so the rows equal evolve.sweep's exactly; rank 0 writes ``out``."""
    import torch.distributed as dist
    from .evolve import GAConfig, sweep_row, sweep_runs, write_sweep_json
    runner = runner or sweep_runs
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    base = base or GAConfig()
    cfgs = [GAConfig(**{**base.__dict__, "mu_L": float(mu)}) for mu in mu_L_grid]
    mine = []
    for i, cfg in enumerate(cfgs):
        seeds = [seed0 + r for r in range(rank, runs, world)]
        recs = runner(cfg, seeds) if seeds else []
        mine.append([(s, rec.discovery, rec.adaptation) for s, rec in zip(seeds, recs)])
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    rows = []
    for i, (mu, cfg) in enumerate(zip(mu_L_grid, cfgs)):
        got = sorted((t for p in parts for t in p[i]), key=lambda t: t[0])
        if [t[0] for t in got] != [seed0 + r for r in range(runs)]:
            raise RuntimeError("sweep_distributed: runs missing after the gather")
        rows.append(sweep_row(mu, cfg, [t[1] for t in got], [t[2] for t in got], sample_size, resamples))
    if out is not None and rank == 0:
        write_sweep_json(out, rows, base, seed0=seed0, sample_size=sample_size, resamples=resamples)
    return rows


def rank_chunks(plan: list, rank: int, world: int) -> list:
    """Round-robin assignment of enumeration chunks to ranks."""
    return [c for i, c in enumerate(plan) if i % world == rank]


def enumerate_space_distributed(space, d: int = 19, k: int = 8, seed: int = 0, batch_size: int = 1 << 20, *,
                                ks=None, hist_k: int | None = None, strict: bool = True, start: int = 0,
                                count: int | None = None, capacity: int = 1 << 20, group=None,
                                device_exchange: bool | None = None) -> Histogram:
    """enumerate_space over all ranks of ``group`` (one GPU per rank).  The exchange is the
    device-resident one (allreduce_device_histogram) on NCCL, the host one otherwise;
    ``device_exchange`` overrides that choice (tests run the device merge over gloo)."""
    import torch.distributed as dist
    ks = tuple(sorted(int(x) for x in (ks if ks is not None else (k,))))
    hist_k = int(hist_k if hist_k is not None else ks[-1])
    if count is None:
        count = space.cardinality - start
    if start < 0 or count < 0 or start + count > space.cardinality:
        raise ValueError(f"[start, start+count) = [{start}, {start + count}) is outside the space "
                         f"(cardinality {space.cardinality})")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    plan = rank_chunks(chunk_plan(start, count, batch_size), rank, world)
    dev = DeviceHistogram(ks, hist_k, shape_words_for(d), capacity)
    try:
        # register the enumeration parameters on every rank, also one with no chunks: after the
        # exchange it owns keys whose payloads may need the export's re-derivation
        dev.enumerate_range(space, start, 0, d, seed, strict)
        # the rank's full chunks in one strided launch (one kernel tail), a partial last chunk apart
        full = [(s, n) for s, n in plan if n == batch_size]
        if full:
            dev.enumerate_chunks(space, full[0][0], len(full) * batch_size, batch_size, batch_size * world, d, seed,
                                 strict)
        for s, n in plan:
            if n != batch_size:
                dev.enumerate_range(space, s, n, d, seed, strict)
        if device_exchange is None:
            device_exchange = dist.get_backend(group) == "nccl"
        if device_exchange:
            out = allreduce_device_histogram(dev, group, meta=_space_meta(space, d, seed, strict))
        else:
            out = allreduce_histogram(dev.export(meta=_space_meta(space, d, seed, strict)), group)
    finally:
        dev.close()
    out.meta.update(start=int(start), count=int(count), world=world)
    return out
