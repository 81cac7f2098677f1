"""GPU edge cases of the C-ABI paths: empty inputs, capacity limits, parameter
mismatches, hist_k < ks[-1] in histogram mode, device merges that bring a lower
representative, and the last indices of the S32 space."""
import numpy as np
import pytest

from tests import _golden as G

pytestmark = pytest.mark.gpu

S28_ARGS = (2, 3, np.zeros(0, np.int64), np.zeros(0, np.uint8), np.arange(23, -1, -1, dtype=np.int64))


@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available()
    from paper_2205_15311_b200 import _kernels, _lib, classify, genome
    return _kernels, _lib, classify, genome


def test_empty_batch_and_range(M):
    K, L, C, Gm = M
    out = G.fresh_outputs(0, 4)
    K.classify_batch(np.zeros(0, np.uint64), *S28_ARGS, 19, np.array([1, 2, 4, 8]), 8, np.uint64(0), True,
                     *[out[k] for k in G.OUT_KEYS])
    dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 10)
    dh.enumerate_range(Gm.SearchSpace(2, 8), 0x123, 0, 19, 0, True)
    h = dh.export()
    assert len(h) == 0 and h.total == 0


def test_histogram_capacity_overflow_raises(M):
    K, L, C, Gm = M
    dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 16)  # 16 slots < 2,233 S28 phenotypes
    dh.enumerate_range(Gm.SearchSpace(2, 8), 0, 1 << 24, 19, 0, True)
    with pytest.raises(L.TvError):
        dh.export()


def test_histogram_refuses_other_parameters(M):
    K, L, C, Gm = M
    dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 12)
    sp = Gm.SearchSpace(2, 8)
    dh.enumerate_range(sp, 0, 4096, 19, 0, True)
    with pytest.raises(ValueError):
        dh.enumerate_range(sp, 4096, 4096, 19, 1, True)  # different seed
    with pytest.raises(ValueError):
        dh.enumerate_range(sp, 4096, 4096, 19, 0, False)  # different contact rule
    dh.clear()
    dh.enumerate_range(sp, 4096, 4096, 19, 1, True)  # fine after clear
    assert dh.export().total == 4096


@pytest.mark.parametrize("ks,hist_k", [((1, 2, 4, 8), 4), ((2, 8), 2), ((8,), 8), ((1,), 1), ((3,), 3), ((2, 5), 5)])
def test_histogram_mode_hist_k_below_kmax(M, ks, hist_k):
    """Histogram = aggregation of the oracle's per-genome rows for prefix ks with hist_k < ks[-1]."""
    from oracle import oracle as O
    K, L, C, Gm = M
    idx = np.arange(0x5A0000, 0x5A0000 + (1 << 16), dtype=np.uint64)
    o = G.fresh_outputs(idx.shape[0], len(ks))
    O.classify_batch(idx, *S28_ARGS, 19, np.array(ks), hist_k, 0, True, *[o[k] for k in G.OUT_KEYS])
    exp = C.Histogram.from_rows(idx, *[o[k] for k in G.OUT_KEYS], ks=ks, hist_k=hist_k, W=5)
    dh = C.DeviceHistogram(ks, hist_k, 5, 1 << 14)
    dh.enumerate_range(Gm.SearchSpace(2, 8), int(idx[0]), idx.shape[0], 19, 0, True)
    got = dh.export()
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "w", "h", "cells", "tallies"):
        assert np.array_equal(getattr(got, k).astype(np.int64), getattr(exp, k).astype(np.int64)), k
    assert np.array_equal(got.shape, exp.shape)


def test_device_merge_lower_representative_brings_payload(M):
    """A merged record whose rep_any is lower than the device's takes over the payload."""
    K, L, C, Gm = M
    sp = Gm.SearchSpace(2, 8)
    dh = C.DeviceHistogram((1, 2, 4, 8), 8, 5, 1 << 12)
    dh.enumerate_range(sp, 1 << 20, 1 << 16, 19, 0, True)
    h = dh.export()
    i = int(np.argmax(h.det))
    fake = C.Histogram((1, 2, 4, 8), 8, 5, keys=h.keys[i:i + 1].copy(), det=np.array([1], np.uint64),
                       steric=np.zeros(1, np.uint64), rep_det=np.array([5], np.uint64),
                       rep_any=np.array([5], np.uint64), w=np.array([1], np.uint8), h=np.array([1], np.uint8),
                       cells=np.array([1], np.uint16), shape=np.array([[1, 0, 0, 0, 0]], np.uint64),
                       tallies=np.zeros((4, 5), np.int64))
    dh.merge(fake)
    m = dh.export()
    j = int(np.searchsorted(m.keys, h.keys[i]))
    assert int(m.rep_any[j]) == 5 and int(m.det[j]) == int(h.det[i]) + 1
    assert (int(m.w[j]), int(m.h[j]), int(m.cells[j]), int(m.shape[j, 0])) == (1, 1, 1, 1)
    # a record with a higher representative leaves the payload alone
    dh.clear()
    dh.enumerate_range(sp, 1 << 20, 1 << 16, 19, 0, True)
    fake.rep_any[:] = fake.rep_det[:] = np.uint64(1 << 40)
    dh.merge(fake)
    m = dh.export()
    assert (int(m.w[j]), int(m.h[j]), int(m.cells[j])) == (int(h.w[i]), int(h.h[i]), int(h.cells[i]))
    assert np.array_equal(m.shape[j], h.shape[i])


def test_s32_top_of_index_range_vs_oracle(M):
    """The last 2^16 indices of S32 (index bits near 2^32) through classify_batch and the histogram."""
    from oracle import oracle as O
    K, L, C, Gm = M
    sp = Gm.space_from_preset("s32_3_8")
    a, bpl, mp, mv, fp = sp.kernel_args()
    idx = np.arange((1 << 32) - (1 << 16), 1 << 32, dtype=np.uint64)
    g = G.fresh_outputs(idx.shape[0], 1)
    o = G.fresh_outputs(idx.shape[0], 1)
    K.classify_batch(idx, a, bpl, mp, mv, fp, 19, np.array([7]), 7, np.uint64(0), True, *[g[k] for k in G.OUT_KEYS])
    O.classify_batch(idx, a, bpl, mp, mv, fp, 19, np.array([7]), 7, 0, True, *[o[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert np.array_equal(g[k], o[k]), k
    h = C.enumerate_space(sp, ks=(7,), start=int(idx[0]), count=idx.shape[0], batch_size=1 << 14)
    exp = C.Histogram.from_rows(idx, *[o[k] for k in G.OUT_KEYS], ks=(7,), hist_k=7, W=5)
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "w", "h", "cells", "tallies"):
        assert np.array_equal(getattr(h, k).astype(np.int64), getattr(exp, k).astype(np.int64)), k


def test_spec_acceptance_2_s28_reference_values(M):
    """SPEC ACCEPTANCE 2 on the device, against the reference's own S_{2,8} values recorded in
    SURVEY.md section 0 (71 hashes with DET and STERIC genomes, steric/unbound = 0.124,
    106 DET hashes) and the monotone misclassification (c) relative to k = 32."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "acc", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "acceptance_s28.py"))
    acc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(acc)
    r = acc.run()
    assert r["a_mixed_hashes"] == 71 and r["det_hashes"] == 106
    assert abs(r["b_steric_over_unbound_k8"] - 0.124) < 0.0005
    assert r["c_non_increasing"] and r["c_misclassified_det_vs_k32"]["32"] == 0.0
    hg = G.hist_golden("s28_full")  # prefix tallies at k <= 8 equal the reference's
    for i, k in enumerate((1, 2, 4, 8)):
        t = r["tallies"][str(k)]
        assert [t["det"], t["trivial"], t["steric"], t["unbound"], t["error"]] == hg["tallies"][i].tolist()


def test_spec_acceptance_3_s28_hash_integrity(M):
    """No two distinct deterministic S_{2,8} shapes share a 32-bit hash (SPEC ACCEPTANCE 3)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "hi", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "hash_integrity.py"))
    hi = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(hi)
    r = hi.run("s28")
    assert r["det_payloads"] == r["det_hashes"] == 106 and r["colliding_hashes"] == 0
    assert f"{r['collision_probability_1000'] * 100:.1g}" == "0.01"  # Eq. 2: ~0.01 % for 1000 phenotypes


def test_spec_acceptance_7_csv_byte_identical(M):
    """Same (seed, k, d, space) with different batch sizes and chunk orders -> byte-identical CSV."""
    K, L, C, Gm = M
    sp = Gm.SearchSpace(2, 8)
    a = C.enumerate_space(sp, ks=(1, 2, 4, 8), start=0x300000, count=1 << 19, batch_size=1 << 19).to_csv()
    b = C.enumerate_space(sp, ks=(1, 2, 4, 8), start=0x300000, count=1 << 19, batch_size=12345).to_csv()
    plan = C.chunk_plan(0x300000, 1 << 19, 1 << 15)[::-1]  # reversed chunk order
    c = C.enumerate_space(sp, ks=(1, 2, 4, 8), start=0x300000, count=1 << 19, chunks=plan).to_csv()
    assert a.encode() == b.encode() == c.encode()


@pytest.mark.parametrize("space,ks,chunk", [("s28", (1, 2, 4, 8), 1 << 18), ("s32", (7,), 1 << 20)])
def test_device_exchange_rows_equal_single_histogram(M, space, ks, chunk):
    """The multi-GPU exchange on one GPU: R 'ranks' enumerate round-robin chunks into their own
    device histograms, pack raw rows (payload = claimer, no fix-up), and one histogram merges
    all rows (tv_hist_replace_rows) -> its export equals the single-histogram enumeration,
    payloads included (lowest owner wins, stale payloads re-derived at export)."""
    import torch
    K, L, C, Gm = M
    sp = Gm.SearchSpace(2, 8) if space == "s28" else Gm.space_from_preset("s32_3_8")
    start, count, R = (0, 1 << 22, 3) if space == "s28" else (0x9E370000, 1 << 22, 4)
    plan = C.chunk_plan(start, count, chunk)
    full = C.DeviceHistogram(ks, ks[-1], 5, 1 << 20)
    for s, n in plan:
        full.enumerate_range(sp, s, n, 19, 0, True)
    exp = full.export()
    parts = []
    for r in range(R):
        dh = C.DeviceHistogram(ks, ks[-1], 5, 1 << 20)
        for s, n in plan[r::R]:
            dh.enumerate_range(sp, s, n, 19, 0, True)
        parts.append(dh)
    rows, tal = [], torch.zeros((len(ks), 5), dtype=torch.int64, device="cuda")
    for dh in parts:
        n = dh.count()[0]
        rr = torch.zeros((n + 7, dh.row_width), dtype=torch.int64, device="cuda")  # + padding rows
        t = torch.zeros((len(ks), 5), dtype=torch.int64, device="cuda")
        assert dh.pack_into(rr, t) == n
        rows.append(rr)
        tal += t
    parts[1].replace_rows(torch.cat(rows), tal)
    got = parts[1].export()
    assert got == exp


@pytest.mark.parametrize("d", [41, 97])
def test_histogram_mode_large_grid_vs_oracle(M, d):
    """Histogram mode on large grids (fewer lanes per CTA, wide shape rows) equals the
    aggregation of the oracle's per-genome rows."""
    from oracle import oracle as O
    K, L, C, Gm = M
    idx = np.arange(0x71000, 0x71000 + (1 << 13), dtype=np.uint64)
    W = ((d - 2) ** 2 + 63) // 64
    ks = (1, 2, 4)
    o = G.fresh_outputs(idx.shape[0], len(ks), W)
    O.classify_batch(idx, *S28_ARGS, d, np.array(ks), 4, 0, True, *[o[k] for k in G.OUT_KEYS])
    exp = C.Histogram.from_rows(idx, *[o[k] for k in G.OUT_KEYS], ks=ks, hist_k=4, W=W)
    dh = C.DeviceHistogram(ks, 4, W, 1 << 14)
    dh.enumerate_range(Gm.SearchSpace(2, 8), int(idx[0]), idx.shape[0], d, 0, True)
    got = dh.export()
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "w", "h", "cells", "tallies"):
        assert np.array_equal(getattr(got, k).astype(np.int64), getattr(exp, k).astype(np.int64)), k
    assert np.array_equal(got.shape, exp.shape)


def test_generic_kernel_large_grid_vs_oracle(M):
    """d = 151 (generic kernel: beyond the bitboard's shared-memory board) equals the oracle."""
    from oracle import oracle as O
    K, L, C, Gm = M
    d = 151
    idx = np.arange(0x3A0000, 0x3A0000 + 96, dtype=np.uint64)
    W = ((d - 2) ** 2 + 63) // 64
    g = G.fresh_outputs(idx.shape[0], 2, W)
    o = G.fresh_outputs(idx.shape[0], 2, W)
    K.classify_batch(idx, *S28_ARGS, d, np.array([1, 3]), 3, np.uint64(5), False, *[g[k] for k in G.OUT_KEYS])
    assert L.launch_info()["path"] == "generic"
    O.classify_batch(idx, *S28_ARGS, d, np.array([1, 3]), 3, 5, False, *[o[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert np.array_equal(g[k], o[k]), k


@pytest.mark.parametrize("strict", [False, True])
def test_s32_random_nonstrict_and_strict_vs_oracle(M, strict):
    """a = 3 (64-bit candidate planes) under both contact rules, 4096 random S32 genomes, k up to 8."""
    from oracle import oracle as O
    K, L, C, Gm = M
    sp = Gm.space_from_preset("s32_3_8")
    a, bpl, mp, mv, fp = sp.kernel_args()
    idx = np.sort(np.random.default_rng(32 + strict).choice(1 << 32, 4096, replace=False)).astype(np.uint64)
    ks = np.array([1, 4, 8])
    g = G.fresh_outputs(idx.shape[0], 3)
    o = G.fresh_outputs(idx.shape[0], 3)
    K.classify_batch(idx, a, bpl, mp, mv, fp, 19, ks, 8, np.uint64(99), strict, *[g[k] for k in G.OUT_KEYS])
    O.classify_batch(idx, a, bpl, mp, mv, fp, 19, ks, 8, 99, strict, *[o[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert np.array_equal(g[k], o[k]), k


def test_histogram_mode_a1_full_space_vs_oracle(M):
    """a = 1: the whole S_{1,8} (4096 genomes) into the device histogram with k = 16 prefixes."""
    from oracle import oracle as O
    K, L, C, Gm = M
    sp = Gm.SearchSpace(1, 8)
    a, bpl, mp, mv, fp = sp.kernel_args()
    idx = np.arange(sp.cardinality, dtype=np.uint64)
    ks = (1, 2, 4, 8, 16)
    o = G.fresh_outputs(idx.shape[0], len(ks), 5)
    O.classify_batch(idx, a, bpl, mp, mv, fp, 19, np.array(ks), 16, 0, True, *[o[k] for k in G.OUT_KEYS])
    exp = C.Histogram.from_rows(idx, *[o[k] for k in G.OUT_KEYS], ks=ks, hist_k=16, W=5)
    dh = C.DeviceHistogram(ks, 16, 5, 1 << 12)
    dh.enumerate_range(sp, 0, sp.cardinality, 19, 0, True)
    got = dh.export()
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "w", "h", "cells", "tallies"):
        assert np.array_equal(getattr(got, k).astype(np.int64), getattr(exp, k).astype(np.int64)), k
    assert np.array_equal(got.shape, exp.shape)


@pytest.mark.parametrize("d", [61, 181])
def test_single_genome_apis_large_grid_vs_oracle(M, d):
    """classify_single / assemble_single (one device thread) on large grids: line-prone tile
    sets grow long runs; every return value, the shape words and the grid equal the oracle."""
    from oracle import oracle as O
    K, L, C, Gm = M
    rng = np.random.default_rng(d)
    W = ((d - 2) ** 2 + 63) // 64
    for t in range(12):
        labels = rng.integers(0, 8, 8).astype(np.uint8)
        labels[2] = ((labels[0] - 1) ^ 1) + 1 if labels[0] else 1  # tile 0 bonds itself N-S: long runs
        e = K.edges_from_labels(labels, 2)
        sw_g, sw_o = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
        assert K.classify_single(e, 2, d, 4, 7, t, True, sw_g) == O.classify_single(e, 2, d, 4, 7, t, True, sw_o)
        assert np.array_equal(sw_g, sw_o)
        gg, go = np.empty(d * d, np.int16), np.empty(d * d, np.int16)
        assert K.assemble_single(e, 2, d, 7, t, 1, False, gg) == O.assemble_single(e, 2, d, 7, t, 1, False, go)
        assert np.array_equal(gg, go)
