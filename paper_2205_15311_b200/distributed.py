"""Multi-GPU enumeration: index-range sharding plus one histogram exchange.

Enumeration shards naturally -- every genome's substream is keyed by
(seed, enumeration index, run) (_k:45-48), so which rank processes an index
cannot change its result.  Chunks are dealt round-robin (chunk c -> rank
c mod R) because work varies strongly with the high index bits (the seed
tile's labels).  The only exchange is at the end: the per-rank histograms are
combined by ``allreduce_histogram`` -- an all-gather of the (tiny) key sets to
build the same sorted key union on every rank, then dense all-reduces over
that union: SUM for counts and class tallies, MIN for representatives, then
MAX over the payloads where only the rank holding the representative (lowest
rep_any) contributes, so colliding shapes under one hash resolve exactly as
the per-genome aggregation does.  With the NCCL backend the
tensors live in HBM and the collectives run over NVLink; the same code runs on
gloo/CPU for the multi-process tests.
"""
from __future__ import annotations

import numpy as np

from .classify import DeviceHistogram, Histogram, _space_meta, chunk_plan, shape_words_for  # noqa: F401

I64_MAX = np.iinfo(np.int64).max
I64_MIN = np.iinfo(np.int64).min
U64_MAX = np.iinfo(np.uint64).max


def _dev(group):
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def allreduce_histogram(h: Histogram, group=None) -> Histogram:
    """Combine per-rank histograms; every rank returns the identical merged result."""
    import torch
    import torch.distributed as dist

    dev = _dev(group)
    world = dist.get_world_size(group)
    n = torch.tensor([len(h)], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    nmax = max(int(x.item()) for x in ns)
    kp = torch.full((max(nmax, 1),), -1, dtype=torch.int64, device=dev)
    if len(h):
        kp[: len(h)] = torch.from_numpy(h.keys.astype(np.int64)).to(dev)
    allk = [torch.empty_like(kp) for _ in range(world)]
    dist.all_gather(allk, kp, group=group)
    union = torch.unique(torch.cat(allk))
    union = union[union >= 0]
    U = int(union.numel())
    pos = torch.searchsorted(union, torch.from_numpy(h.keys.astype(np.int64)).to(dev))
    q5 = h.tallies.size
    sums = torch.zeros(2 * U + q5, dtype=torch.int64, device=dev)
    sums[pos] = torch.from_numpy(h.det.astype(np.int64)).to(dev)
    sums[U + pos] = torch.from_numpy(h.steric.astype(np.int64)).to(dev)
    sums[2 * U:] = torch.from_numpy(h.tallies.reshape(-1).astype(np.int64)).to(dev)
    mins = torch.full((2 * U,), I64_MAX, dtype=torch.int64, device=dev)

    def rep(a):
        r = a.astype(np.uint64)
        return torch.from_numpy(np.where(r == U64_MAX, I64_MAX, r.astype(np.int64))).to(dev)
    mins[pos] = rep(h.rep_det)
    mins[U + pos] = rep(h.rep_any)
    W = h.W
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mins, op=dist.ReduceOp.MIN, group=group)
    # payload = the representative's (lowest rep_any): only the rank holding it contributes
    maxs = torch.full((U, 1 + W), I64_MIN, dtype=torch.int64, device=dev)
    whc = h.w.astype(np.int64) | (h.h.astype(np.int64) << 8) | (h.cells.astype(np.int64) << 16)
    own = rep(h.rep_any) == mins[U + pos]
    maxs[pos[own], 0] = torch.from_numpy(whc).to(dev)[own]
    maxs[pos[own], 1:] = torch.from_numpy(np.ascontiguousarray(h.shape).view(np.int64)).to(dev)[own]
    dist.all_reduce(maxs, op=dist.ReduceOp.MAX, group=group)
    s = sums.cpu().numpy()
    m = mins.cpu().numpy()
    x = maxs.cpu().numpy()
    out = Histogram(h.ks, h.hist_k, W, meta=dict(h.meta))
    out.keys = union.cpu().numpy().astype(np.uint32)
    out.det = s[:U].astype(np.uint64)
    out.steric = s[U:2 * U].astype(np.uint64)
    out.tallies = s[2 * U:].reshape(h.tallies.shape).astype(np.int64)

    def unrep(a):
        return np.where(a == I64_MAX, U64_MAX, a.astype(np.uint64)).astype(np.uint64)
    out.rep_det = unrep(m[:U])
    out.rep_any = unrep(m[U:])
    out.w = (x[:, 0] & 0xFF).astype(np.uint8)
    out.h = ((x[:, 0] >> 8) & 0xFF).astype(np.uint8)
    out.cells = ((x[:, 0] >> 16) & 0xFFFF).astype(np.uint16)
    out.shape = np.ascontiguousarray(x[:, 1:]).view(np.uint64).reshape(U, W)
    return out


def allreduce_device_histogram(dev: DeviceHistogram, group=None, meta: dict | None = None,
                               export: bool = True) -> Histogram | None:
    """Device-resident exchange (NCCL): every rank packs its raw records on the GPU, one
    all_gather moves them over NVLink, one all_reduce sums the tallies, and each rank
    merges all rows into its own device histogram (tv_hist_replace_rows: counts added,
    representatives lowered, payload = lowest owner) before the export re-derives the
    payloads whose owner is not the representative.  Same result as allreduce_histogram.
    export=False stops with the merged histogram resident in ``dev`` (returns None)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n_local, _ = dev.count()
    dv = torch.device("cuda", torch.cuda.current_device())
    # collectives on the device for NCCL; other backends (gloo: several ranks sharing one GPU
    # in tests) move the same tensors through host memory
    cv = dv if dist.get_backend(group) == "nccl" else torch.device("cpu")
    nmax = torch.tensor([n_local], dtype=torch.int64, device=cv)
    dist.all_reduce(nmax, op=dist.ReduceOp.MAX, group=group)
    nmax = max(1, int(nmax.item()))
    rows = torch.zeros((nmax, dev.row_width), dtype=torch.int64, device=dv)
    tallies = torch.zeros((len(dev.ks), 5), dtype=torch.int64, device=dv)
    dev.pack_into(rows, tallies)
    allrows = torch.empty((world * nmax, dev.row_width), dtype=torch.int64, device=cv)
    rows_c, tallies_c = rows.to(cv), tallies.to(cv)
    dist.all_gather_into_tensor(allrows, rows_c, group=group)
    dist.all_reduce(tallies_c, op=dist.ReduceOp.SUM, group=group)
    dev.replace_rows(allrows.to(dv), tallies_c.to(dv))
    return dev.export(meta=meta) if export else None


def rank_chunks(plan: list, rank: int, world: int) -> list:
    """Round-robin assignment of enumeration chunks to ranks."""
    return [c for i, c in enumerate(plan) if i % world == rank]


def enumerate_space_distributed(space, d: int = 19, k: int = 8, seed: int = 0, batch_size: int = 1 << 20, *,
                                ks=None, hist_k: int | None = None, strict: bool = True, start: int = 0,
                                count: int | None = None, capacity: int = 1 << 20, group=None) -> Histogram:
    """enumerate_space over all ranks of ``group`` (one GPU per rank)."""
    import torch.distributed as dist
    ks = tuple(sorted(int(x) for x in (ks if ks is not None else (k,))))
    hist_k = int(hist_k if hist_k is not None else ks[-1])
    if count is None:
        count = space.cardinality - start
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    plan = rank_chunks(chunk_plan(start, count, batch_size), rank, world)
    dev = DeviceHistogram(ks, hist_k, shape_words_for(d), capacity)
    try:
        # the rank's full chunks in one strided launch (one kernel tail), a partial last chunk apart
        full = [(s, n) for s, n in plan if n == batch_size]
        if full:
            dev.enumerate_chunks(space, full[0][0], len(full) * batch_size, batch_size, batch_size * world, d, seed,
                                 strict)
        for s, n in plan:
            if n != batch_size:
                dev.enumerate_range(space, s, n, d, seed, strict)
        if dist.get_backend(group) == "nccl":
            out = allreduce_device_histogram(dev, group, meta=_space_meta(space, d, seed, strict))
        else:
            out = allreduce_histogram(dev.export(meta=_space_meta(space, d, seed, strict)), group)
    finally:
        dev.close()
    out.meta.update(start=int(start), count=int(count), world=world)
    return out
