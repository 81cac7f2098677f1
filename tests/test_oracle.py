"""Pin the CPU restatement (oracle/) to the reference's golden vectors.

The oracle is the checker for every GPU parity test, so it must itself be
bit-exact with the reference: fixtures in tests/golden/ were produced by
running /root/reference (tilevolve, numba) -- see make_golden.py -- and the
large-range digests also equal SURVEY.md Appendix C.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests import _golden as G


def test_oat_vectors():
    for data, h in G.vectors()["oat"]:
        assert O.oat_hash_bytes(np.array(data, np.uint8)) == h


def test_oat_spec_examples():
    # SPEC.md:249 (empty -> 0) and SURVEY.md section 4 pinned values
    assert O.oat_hash_bytes(np.zeros(0, np.uint8)) == 0
    assert O.oat_hash_bytes(np.array([0x61], np.uint8)) == 0xCA2E9442
    assert O.oat_hash_bytes(np.array([1, 2, 3], np.uint8)) == 0xF926DA4F
    assert O.oat_hash_bytes(np.array([1, 1, 0, 0], np.uint8)) == 0x3A9BE4CF


def test_rng_streams():
    for s in G.vectors()["streams"]:
        got = O.stream_draws(s["seed"], s["idx"], s["run"], 16)
        assert [int(x) for x in got] == [int(x) for x in s["draws"]]
        # bounded draws use the high word: ((x >> 32) * n) >> 32
        bel = [((int(x) >> 32) * n) >> 32 for x, n in zip(got, (2, 3, 4, 2, 3, 4, 5, 7))]
        assert bel == s["below"]


def _edges(tiles):
    from paper_2205_15311_b200._kernels import edges_from_labels
    return edges_from_labels(np.array([v for t in tiles for v in t], np.uint8), len(tiles))


def test_classify_single_vectors():
    for c in G.vectors()["classify_single"]:
        d = c["d"]
        sw = np.full((d * d + 63) // 64, 0xAB, np.uint64)
        res = O.classify_single(_edges(c["tiles"]), len(c["tiles"]), d, c["k"], c["seed"], c["genome_index"],
                                c["strict"], sw)
        assert list(res) == c["result"], c
        assert [int(x) for x in sw] == [int(x) for x in c["shape"]], c


def test_assemble_single_vectors():
    for c in G.vectors()["assemble_single"]:
        d = c["d"]
        g = np.empty(d * d, np.int16)
        res = O.assemble_single(_edges(c["tiles"]), len(c["tiles"]), d, 0, c["genome_index"], c["run"], True, g)
        assert list(res) == c["result"], c
        assert g.tolist() == c["grid"], c


@pytest.mark.parametrize("name", G.slice_names())
def test_classify_batch_slices(name):
    c = G.slice_case(name)
    n = c["idx"].shape[0]
    out = G.fresh_outputs(n, len(c["ks"]), prefill=c["prefill"])
    O.classify_batch(c["idx"], c["a"], c["bpl"], c["mp"], c["mv"], c["free"], c["d"], np.array(c["ks"]),
                     c["hist_k"], c["seed"], c["strict"], *[out[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert np.array_equal(out[k], c["expected"][k]), (name, k)


@pytest.mark.parametrize("name", ["s28_1m", "s32_1m"])
def test_large_slice_digests_and_histogram(name):
    dg = G.digests()[name]
    ks = dg["ks"]
    if name.startswith("s28"):
        a, bpl, mp, mv, free = 2, 3, np.zeros(0, np.int64), np.zeros(0, np.uint8), np.arange(23, -1, -1)
    else:
        a, bpl, mp, mv, free = 3, 3, np.array([32, 33, 34, 35]), np.zeros(4, np.uint8), np.arange(31, -1, -1)
    idx = np.arange(dg["start"], dg["start"] + dg["n"], dtype=np.uint64)
    out = G.fresh_outputs(idx.shape[0], len(ks))
    O.classify_batch(idx, a, bpl, mp, mv, free, 19, np.array(ks), ks[-1], 0, True, *[out[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert G.sha(out[k]) == dg["digests"][k], (name, k)
    hg = G.hist_golden(name)
    mine = G.histogram_from_outputs(out, idx, ks, ks[-1])
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "tallies"):
        assert np.array_equal(mine[k].astype(np.int64), hg[k].astype(np.int64)), k


def test_survey_digests_pinned():
    """The reference digests we regenerated equal SURVEY.md Appendix C."""
    dg = G.digests()
    assert dg["s28_1m"]["digests"]["cls"].startswith("d80e1d0d76951088")
    assert dg["s28_full"]["digests"]["shape"].startswith("80bb1eb2e5a6bbcb")
    assert dg["s32_1m"]["digests"]["hash"].startswith("d313fa1ff6789e42")


@pytest.mark.slow
def test_full_s28_digests():
    dg = G.digests()["s28_full"]
    idx = np.arange(0, 1 << 24, dtype=np.uint64)
    out = G.fresh_outputs(idx.shape[0], 4)
    O.classify_batch(idx, 2, 3, np.zeros(0, np.int64), np.zeros(0, np.uint8), np.arange(23, -1, -1), 19,
                     np.array([1, 2, 4, 8]), 8, 0, True, *[out[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert G.sha(out[k]) == dg["digests"][k], k


@pytest.mark.parametrize("kind", ["blocks", "random"])
def test_s32_reference_samples(kind):
    """The oracle equals the REFERENCE (numba) on 4.2 M S32 genomes spread over the whole
    2^32 index range (tests/golden/make_s32_sample.py): every output column's digest and
    the histogram aggregate."""
    idx, meta = G.s32_sample(kind)
    a, bpl, mp, mv, free = 3, 3, np.array([32, 33, 34, 35]), np.zeros(4, np.uint8), np.arange(31, -1, -1)
    out = G.fresh_outputs(idx.shape[0], 1)
    O.classify_batch(idx, a, bpl, mp, mv, free, 19, np.array([7]), 7, 0, True, *[out[k] for k in G.OUT_KEYS])
    for k in G.OUT_KEYS:
        assert G.sha(out[k]) == meta["digests"][k], (kind, k)
    hg = G.hist_golden("s32_" + kind)
    mine = G.histogram_from_outputs(out, idx, [7], 7)
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "tallies"):
        assert np.array_equal(mine[k].astype(np.int64), hg[k].astype(np.int64)), k
