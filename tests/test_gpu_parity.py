"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
fixtures and the pinned CPU oracle.  Bit-exact for every output column."""
import numpy as np
import pytest

from tests import _golden as G

pytestmark = pytest.mark.gpu

S28_ARGS = (2, 3, np.zeros(0, np.int64), np.zeros(0, np.uint8), np.arange(23, -1, -1, dtype=np.int64))
S32_ARGS = (3, 3, np.array([32, 33, 34, 35], np.int64), np.zeros(4, np.uint8), np.arange(31, -1, -1, dtype=np.int64))


@pytest.fixture(scope="module")
def K():
    import torch
    assert torch.cuda.is_available(), "GPU test needs CUDA"
    from paper_2205_15311_b200 import _kernels
    return _kernels


def _run(K, c, out):
    K.classify_batch(c["idx"], c["a"], c["bpl"], c["mp"], c["mv"], c["free"], c["d"], np.array(c["ks"]),
                     c["hist_k"], np.uint64(c["seed"]), c["strict"], *[out[k] for k in G.OUT_KEYS])


@pytest.mark.parametrize("name", G.slice_names())
def test_classify_batch_golden_slices(K, name):
    c = G.slice_case(name)
    out = G.fresh_outputs(c["idx"].shape[0], len(c["ks"]), prefill=c["prefill"])
    _run(K, c, out)
    for k in G.OUT_KEYS:
        assert np.array_equal(out[k], c["expected"][k]), (name, k)


def test_classify_batch_device_tensors(K):
    import torch
    c = G.slice_case("s28_rand")
    n = c["idx"].shape[0]
    exp = c["expected"]
    dev = dict(cls=torch.zeros((n, 4), dtype=torch.uint8, device="cuda"),
               hash=torch.zeros(n, dtype=torch.uint32, device="cuda"),
               w=torch.zeros(n, dtype=torch.uint8, device="cuda"), h=torch.zeros(n, dtype=torch.uint8, device="cuda"),
               cells=torch.zeros(n, dtype=torch.uint16, device="cuda"),
               shape=torch.zeros((n, 6), dtype=torch.uint64, device="cuda"))
    idx = torch.from_numpy(c["idx"].astype(np.int64)).to("cuda").view(torch.uint64)
    K.classify_batch(idx, c["a"], c["bpl"], c["mp"], c["mv"], c["free"], 19, np.array(c["ks"]), c["hist_k"],
                     np.uint64(0), True, *[dev[k] for k in G.OUT_KEYS])
    torch.cuda.synchronize()
    for k in G.OUT_KEYS:
        got = dev[k].cpu().numpy()
        assert np.array_equal(got, exp[k]), k


def test_launch_path_is_bitboard_kernel(K):
    from paper_2205_15311_b200 import _lib
    c = G.slice_case("s28_800000")
    out = G.fresh_outputs(c["idx"].shape[0], 4)
    _run(K, c, out)
    info = _lib.launch_info()
    assert info["path"] == "bitboard" and info["launches"] >= 1, info
    c = G.slice_case("s48_rand")  # a=4 -> generic kernel
    out = G.fresh_outputs(c["idx"].shape[0], len(c["ks"]))
    _run(K, c, out)
    assert _lib.launch_info()["path"] == "generic"


def _edges(tiles):
    from paper_2205_15311_b200._kernels import edges_from_labels
    return edges_from_labels(np.array([v for t in tiles for v in t], np.uint8), len(tiles))


def test_classify_single_vectors(K):
    for c in G.vectors()["classify_single"]:
        d = c["d"]
        sw = np.full((d * d + 63) // 64, 0xAB, np.uint64)
        res = K.classify_single(_edges(c["tiles"]), len(c["tiles"]), d, c["k"], c["seed"], c["genome_index"],
                                c["strict"], sw)
        assert [int(x) for x in res] == c["result"], c
        assert [int(x) for x in sw] == [int(x) for x in c["shape"]], c


def test_assemble_single_vectors(K):
    for c in G.vectors()["assemble_single"]:
        d = c["d"]
        g = np.empty(d * d, np.int16)
        res = K.assemble_single(_edges(c["tiles"]), len(c["tiles"]), d, 0, c["genome_index"], c["run"], True, g)
        assert list(res) == c["result"], c
        assert g.tolist() == c["grid"], c


def test_oat_hash_bytes(K):
    for data, h in G.vectors()["oat"]:
        assert int(K.oat_hash_bytes(np.array(data, np.uint8))) == h


@pytest.mark.parametrize("name,args", [("s28_1m", S28_ARGS), ("s32_1m", S32_ARGS)])
def test_large_slice_digests(K, name, args):
    dg = G.digests()[name]
    ks = dg["ks"]
    idx = np.arange(dg["start"], dg["start"] + dg["n"], dtype=np.uint64)
    out = G.fresh_outputs(idx.shape[0], len(ks))
    K.classify_batch(idx, *args, 19, np.array(ks), ks[-1], np.uint64(0), True, *[out[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert G.sha(out[k]) == dg["digests"][k], (name, k)


@pytest.mark.parametrize("kind", ["blocks", "random"])
def test_s32_reference_samples(K, kind):
    """S32 pinned directly to the REFERENCE (numba) at scale: 4.2 M genomes over the whole
    2^32 index range (bench.py's 64 x 2^16 blocks; 2^22 random indices), every per-genome
    output column by SHA-256, and the device histogram of the same indices vs the
    reference aggregate (tests/golden/make_s32_sample.py)."""
    from paper_2205_15311_b200.classify import DeviceHistogram
    from paper_2205_15311_b200.genome import space_from_preset
    idx, meta = G.s32_sample(kind)
    out = G.fresh_outputs(idx.shape[0], 1)
    K.classify_batch(idx, *S32_ARGS, 19, np.array([7]), 7, np.uint64(0), True, *[out[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert G.sha(out[k]) == meta["digests"][k], (kind, k)
    dev = DeviceHistogram((7,), 7, 5, 1 << 16)
    dev.enumerate_indices(space_from_preset("s32_3_8"), idx[::-1].copy(), 19, 0, True)  # any order
    h = dev.export()
    dev.close()
    _check_hist(h, "s32_" + kind)
    assert len(h) == meta["n_keys"]


def test_random_s32_vs_oracle(K):
    """2^20 random S32 indices, GPU vs the pinned oracle (all host threads)."""
    from oracle import oracle as O
    rng = np.random.default_rng(7)
    idx = rng.integers(0, 1 << 32, 1 << 20, dtype=np.uint64)
    a = G.fresh_outputs(idx.shape[0], 1)
    b = G.fresh_outputs(idx.shape[0], 1)
    K.classify_batch(idx, *S32_ARGS, 19, np.array([7]), 7, np.uint64(3), True, *[a[k] for k in G.OUT_KEYS])
    O.classify_batch(idx, *S32_ARGS, 19, np.array([7]), 7, 3, True, *[b[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert np.array_equal(a[k], b[k]), k


def _check_hist(h, name):
    hg = G.hist_golden(name)
    assert np.array_equal(h.keys, hg["keys"])
    for k in ("det", "steric", "rep_det", "rep_any", "tallies"):
        assert np.array_equal(getattr(h, k).astype(np.int64), hg[k].astype(np.int64)), k
    for k in ("w", "h", "cells"):
        assert np.array_equal(getattr(h, k), hg[k]), k
    assert np.array_equal(h.shape[:, :5], hg["shape"][:, :5])


def test_enumerate_full_s28_histogram(K):
    from paper_2205_15311_b200.classify import enumerate_space
    from paper_2205_15311_b200.genome import SearchSpace
    h = enumerate_space(SearchSpace(2, 8), d=19, ks=(1, 2, 4, 8), seed=0, batch_size=1 << 24)
    _check_hist(h, "s28_full")
    assert len(h) == 2233 and int(np.count_nonzero(h.det)) == 106


def test_enumerate_s32_slice_histogram_batch_independent(K):
    from paper_2205_15311_b200.classify import enumerate_space
    from paper_2205_15311_b200.genome import space_from_preset
    sp = space_from_preset("s32_3_8")
    h1 = enumerate_space(sp, ks=(7,), start=0x9E370000, count=1 << 20, batch_size=1 << 20)
    h2 = enumerate_space(sp, ks=(7,), start=0x9E370000, count=1 << 20, batch_size=12345)
    _check_hist(h1, "s32_1m")
    assert h1 == h2


def test_enumerate_generic_path_histogram(K):
    """S_{4,8} sample: generic kernel histogram == aggregation of golden per-genome rows."""
    from paper_2205_15311_b200.classify import DeviceHistogram
    from paper_2205_15311_b200.genome import SearchSpace
    c = G.slice_case("s48_rand")
    dh = DeviceHistogram(c["ks"], c["hist_k"], 5, 1 << 14)
    dh.enumerate_indices(SearchSpace(4, 8), c["idx"], 19, 0, True)
    h = dh.export()
    exp = G.histogram_from_outputs(c["expected"], c["idx"], c["ks"], c["hist_k"])
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "tallies"):
        assert np.array_equal(getattr(h, k).astype(np.int64), exp[k].astype(np.int64)), k


# Exact work elimination switches (read per launch): TV_EARLY_UNBOUND (stop at the first
# UNBOUND run of a provably trivial-free genome), TV_ONEMER (1-mers classified by the
# pre-pass), TV_FORCED (stop after run 0 when its assembly is locally forced).  Results must
# be identical under every combination.
SWITCHES = [(0, 0, 0), (1, 1, 1), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 2)]


@pytest.fixture
def early_unbound(monkeypatch):
    def set_(sw):
        for name, v in zip(("TV_EARLY_UNBOUND", "TV_ONEMER", "TV_FORCED"), sw):
            monkeypatch.setenv(name, str(int(v)))
    return set_


@pytest.mark.parametrize("on", SWITCHES)
def test_early_unbound_cutoff_s28_full(K, early_unbound, on):
    """The cut-offs skip only runs that cannot change a genome's outcome; the full-S28
    histogram must not change under any combination."""
    from paper_2205_15311_b200.classify import enumerate_space
    from paper_2205_15311_b200.genome import SearchSpace
    early_unbound(on)
    h = enumerate_space(SearchSpace(2, 8), d=19, ks=(1, 2, 4, 8), seed=0, batch_size=1 << 24)
    _check_hist(h, "s28_full")


@pytest.mark.parametrize("on", SWITCHES)
def test_early_unbound_cutoff_per_genome(K, early_unbound, on):
    """Per-genome rows (every column, every prefix k) under each switch combination,
    for a = 1, 2, 3 and non-strict contacts, against the pinned oracle."""
    from oracle import oracle as O
    early_unbound(on)
    rng = np.random.default_rng(21)
    cases = [(S28_ARGS, (1, 2, 4, 8), 8, True, 1 << 24), (S32_ARGS, (1, 3, 7), 7, True, 1 << 32),
             (S32_ARGS, (2, 5), 5, False, 1 << 32),
             ((1, 3, np.zeros(0, np.int64), np.zeros(0, np.uint8), np.arange(11, -1, -1, dtype=np.int64)),
              (1, 8), 4, True, 1 << 12)]
    for args, ks, hk, strict, space in cases:
        idx = rng.integers(0, space, 1 << 17, dtype=np.uint64)
        a = G.fresh_outputs(idx.shape[0], len(ks))
        b = G.fresh_outputs(idx.shape[0], len(ks))
        K.classify_batch(idx, *args, 19, np.array(ks), hk, np.uint64(5), strict, *[a[k] for k in G.OUT_KEYS])
        O.classify_batch(idx, *args, 19, np.array(ks), hk, 5, strict, *[b[k] for k in G.OUT_KEYS])
        for k in G.OUT_KEYS:
            assert np.array_equal(a[k], b[k]), (args[0], ks, strict, k)


def test_enumerate_full_s32_histogram(K):
    """All 2^32 S^{32}_{3,8} genomes on one GPU (~10 s) against the oracle's full-space
    aggregate (tests/golden/make_s32_full.py): tallies, key count, per-column SHA-256
    of the sorted records, and the sampled records in full."""
    import hashlib
    import json
    import os
    from paper_2205_15311_b200.classify import enumerate_space
    from paper_2205_15311_b200.genome import space_from_preset
    with open(os.path.join(G.GOLDEN, "hist_s32_full.json")) as f:
        meta = json.load(f)
    smp = dict(np.load(os.path.join(G.GOLDEN, "hist_s32_full_sample.npz")))
    h = enumerate_space(space_from_preset("s32_3_8"), ks=(7,), seed=0, batch_size=1 << 30, capacity=1 << 21)
    assert h.tallies.tolist() == meta["tallies"]
    assert len(h) == meta["n_keys"]
    cols = dict(keys=h.keys.astype(np.uint32), det=h.det.astype(np.uint64), steric=h.steric.astype(np.uint64),
                rep_det=h.rep_det.astype(np.uint64), rep_any=h.rep_any.astype(np.uint64), w=h.w.astype(np.uint8),
                h=h.h.astype(np.uint8), cells=h.cells.astype(np.uint16),
                shape=np.ascontiguousarray(h.shape[:, :5]).astype(np.uint64))
    sel = (cols["keys"] % 64) == 0
    for k, v in cols.items():
        assert np.array_equal(v[sel], smp[k]), k
        assert hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() == meta["sha256"][k], k


@pytest.mark.parametrize("seed,strict", [(2205, True), (7, False)])
def test_enumerate_full_s28_other_seeds_vs_oracle(K, seed, strict):
    """Full S_{2,8} at a seed and contact rule the reference goldens do not cover: device histogram
    (behaviour-sorted order, early cut-off, payload fix-up) == the oracle's per-genome rows
    aggregated on the host, every record column."""
    from oracle import oracle as O
    from paper_2205_15311_b200.classify import Histogram, enumerate_space
    from paper_2205_15311_b200.genome import SearchSpace
    ks = (1, 2, 4, 8)
    h = enumerate_space(SearchSpace(2, 8), d=19, ks=ks, seed=seed, strict=strict, batch_size=1 << 24)
    acc = None
    blk = 1 << 22
    for s in range(0, 1 << 24, blk):
        idx = np.arange(s, s + blk, dtype=np.uint64)
        o = G.fresh_outputs(blk, 4)
        O.classify_batch(idx, *S28_ARGS, 19, np.array(ks), 8, seed, strict, *[o[k] for k in G.OUT_KEYS])
        part = Histogram.from_rows(idx, *[o[k] for k in G.OUT_KEYS], ks=ks, hist_k=8, W=5)
        acc = part if acc is None else acc.merge(part)
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "w", "h", "cells", "tallies"):
        assert np.array_equal(getattr(h, k).astype(np.int64), getattr(acc, k).astype(np.int64)), k
    assert np.array_equal(h.shape, acc.shape)


@pytest.mark.parametrize("d,path", [(61, "bitboard"), (105, "bitboard"), (117, None), (119, "generic")])
def test_large_grid_path_boundary_vs_oracle(K, d, path):
    """Large grids: the bitboard kernel runs while whole warps' boards fit in shared memory
    (fewer lanes per CTA as d grows; d <= 118 for byte cell offsets), beyond that the generic
    kernel; every case equals the oracle row for row (long runs, deep movelists that spill)."""
    from oracle import oracle as O
    from paper_2205_15311_b200 import _lib
    rng = np.random.default_rng(d)
    idx = np.sort(rng.choice(1 << 24, 384, replace=False)).astype(np.uint64)
    args = (2, 3, np.zeros(0, np.int64), np.zeros(0, np.uint8), np.arange(23, -1, -1, dtype=np.int64))
    ks = np.array([1, 2])
    W = ((d - 2) ** 2 + 63) // 64  # shape rows wide enough for the largest crop
    g = G.fresh_outputs(idx.shape[0], 2, W)
    o = G.fresh_outputs(idx.shape[0], 2, W)
    K.classify_batch(idx, *args, d, ks, 2, np.uint64(3), True, *[g[k] for k in G.OUT_KEYS])
    if path is not None:
        assert _lib.launch_info()["path"] == path
    O.classify_batch(idx, *args, d, ks, 2, 3, True, *[o[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert np.array_equal(g[k], o[k]), k
