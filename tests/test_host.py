"""Host-side API parity (CPU): genome codec, assembly helpers, classify utilities,
histogram formats.  Examples are SPEC.md's tagged examples; reference behaviour
is pinned against the golden fixtures where it exists."""
import io
import os

import numpy as np
import pytest

from paper_2205_15311_b200 import assembly as A
from paper_2205_15311_b200 import classify as C
from paper_2205_15311_b200 import genome as G
from tests import _golden as GD


# ---------------------------------------------------------------- genome
def test_decode_examples():
    s = G.SearchSpace(2, 8)
    assert G.decode_tileset(G.Genome(24), s) == G.TileSet(((0, 0, 0, 0), (0, 0, 0, 0)))
    g = G.Genome.from_text("0x200000/24")  # 001 000 ... -> tile0 = (1,0,0,0)
    assert G.decode_tileset(g, s) == G.TileSet(((1, 0, 0, 0), (0, 0, 0, 0)))
    assert G.encode_tileset(G.TileSet(((7, 7, 7, 7), (7, 7, 7, 7))), s).to_int() == (1 << 24) - 1


def test_roundtrips_and_bijectivity():
    rng = np.random.default_rng(1)
    s = G.SearchSpace(2, 8)
    for v in rng.integers(0, 1 << 24, 1000):
        g = G.Genome.from_int(24, int(v))
        assert G.encode_tileset(G.decode_tileset(g, s), s) == g
    s32 = G.space_from_preset("s32_3_8")
    for i in rng.integers(0, 1 << 32, 2000, dtype=np.uint64):
        g = G.genome_at_index(s32, int(i))
        assert G.index_of_genome(s32, g) == int(i)
        assert all(g.bit(p) == 0 for p in (32, 33, 34, 35))
    assert s32.cardinality == 1 << 32 and s32.bit_length == 36


def test_genome_index_matches_reference_decoder_layout():
    """Index -> labels through genome_at_index equals the kernel's decode (golden S32 slice edges)."""
    s32 = G.space_from_preset("s32_3_8")
    i = 0x9E373C1B
    ts = G.decode_tileset(G.genome_at_index(s32, i), s32)
    # unmasked part of an S32 genome read big-endian equals the index's 32 bits
    v = G.genome_at_index(s32, i).to_int()
    assert v >> 4 == i and ts.tiles[2][3] == 0


def test_hamming_and_errors():
    assert G.hamming_weight(G.Genome(32)) == 0
    assert G.hamming_weight(G.Genome.from_int(32, (1 << 32) - 1)) == 32
    assert G.Genome.from_int(16, 0xF0F0).hamming_weight() == 8
    g = G.Genome.from_int(24, 0x123456)
    assert g.hamming_weight() + g.complement().hamming_weight() == 24
    with pytest.raises(G.GenomeError):
        G.SearchSpace(2, 6)
    with pytest.raises(G.GenomeError):
        G.genome_at_index(G.SearchSpace(2, 8), 1 << 24)
    with pytest.raises(G.GenomeError):
        G.Genome.from_text("123/8")
    assert G.Genome.from_text("0x000001/24").to_text() == "0x000001/24"


def test_kernel_args_match_reference_convention():
    a, bpl, mp, mv, fp = G.space_from_preset("s32_3_8").kernel_args()
    c = GD.slice_case("s32_9e37")
    assert (a, bpl) == (c["a"], c["bpl"])
    assert np.array_equal(mp, c["mp"]) and np.array_equal(mv, c["mv"]) and np.array_equal(fp, c["free"])


# ---------------------------------------------------------------- assembly
def test_bonds_examples():
    assert A.bonds(1, 2) and A.bonds(5, 6) and not A.bonds(3, 3)
    assert not any(A.bonds(0, j) for j in range(8))
    assert all(A.bonds(i, j) == A.bonds(j, i) for i in range(8) for j in range(8))


def test_bonding_table_examples():
    bt = A.build_bonding_table(G.TileSet(((0, 0, 0, 0),)), 8)
    assert all(len(e) == 0 for e in bt.entries)
    bt = A.build_bonding_table(G.TileSet(((2, 0, 0, 0), (1, 0, 0, 0))), 8)
    assert [e for e in bt[2] if e[0] == 1] == [(1, 0)]
    bt = A.build_bonding_table(G.TileSet(((1, 1, 1, 1),)), 8)
    assert len(bt[2]) == 1


def test_grid_helpers():
    g = A.AssemblyGrid(5)
    g.cells[2, 2] = 0
    h = A.AssemblyGrid(5, g.cells.copy())
    assert A.outcome_equivalent(g, h) and g.cell(2, 2) == (0, 0) and g.occupied_count() == 1
    with pytest.raises(A.AssemblyError):
        A.outcome_equivalent(g, A.AssemblyGrid(7))
    with pytest.raises(A.AssemblyError):
        A._check_dim(4)


# ---------------------------------------------------------------- classify utilities
def test_oat_and_shape_hash_goldens():
    for data, h in GD.vectors()["oat"]:
        assert C.oat_hash(data) == h
    one = C.CroppedShape(1, 1, np.ones((1, 1), bool))
    assert C.shape_hash(one) == 0x3A9BE4CF
    vdimer = C.CroppedShape(1, 2, np.ones((2, 1), bool))
    assert C.shape_hash(vdimer) == 0xF18EFE69
    hdimer = C.CroppedShape(2, 1, np.ones((1, 2), bool))
    assert C.shape_hash(hdimer) == 0x483F256C


def test_shape_hash_matches_golden_rows():
    c = GD.slice_case("s28_800000")
    e = c["expected"]
    sel = np.nonzero(e["w"])[0][:300]
    for i in sel:
        s = C.CroppedShape.from_packed_words(int(e["w"][i]), int(e["h"][i]), e["shape"][i])
        assert C.shape_hash(s) == int(e["hash"][i])
        assert s.cells == int(e["cells"][i])


def test_rotation_invariant_hash():
    L = C.CroppedShape(2, 3, np.array([[1, 0], [1, 0], [1, 1]], bool))
    J = L.mirrored()
    assert C.shape_hash(L) != C.shape_hash(L.rotated(1))
    assert len({C.rotation_invariant_hash(L.rotated(k)) for k in range(4)}) == 1
    assert C.rotation_invariant_hash(L) != C.rotation_invariant_hash(J)
    assert C.d4_min_hash(L) == C.d4_min_hash(J)
    sq = C.CroppedShape(2, 2, np.ones((2, 2), bool))
    h = C.shape_hash(sq)
    assert C.rotation_invariant_hash(sq) == C.oat_hash(np.frombuffer(np.array([h] * 4, "<u4").tobytes(), np.uint8))


def test_crop_and_shapediff():
    g = A.AssemblyGrid(7)
    g.cells[3, 3] = 0
    g.cells[4, 3] = 1
    s = C.crop(g)
    assert (s.width, s.height, s.cells) == (1, 2, 2)
    h = A.AssemblyGrid(7, g.cells.copy())
    h.cells[3, 4] = 2
    assert C.shapediff(g, h) == 1 == C.shapediff(h, g)
    assert C.shapesim(g, g) == 1.0
    assert abs(C.shapesim(g, h) - (1 - 1 / 49)) < 1e-12


def test_collision_probability():
    assert C.collision_probability(0) == 0.0
    assert abs(C.collision_probability(2) - 2.0 ** -32) < 1e-20
    assert abs(C.collision_probability(1000) - 1.163e-4) < 5e-7


# ---------------------------------------------------------------- histogram formats
def _hist(name="s28_rand"):
    c = GD.slice_case(name)
    e = c["expected"]
    h = C.Histogram.from_rows(c["idx"], e["cls"], e["hash"], e["w"], e["h"], e["cells"], e["shape"], c["ks"],
                              c["hist_k"], W=5, meta=dict(a=2, b=8, fixed_mask=[], d=19, seed=0, strict=True))
    return c, h


def test_from_rows_equals_golden_aggregation():
    c, h = _hist()
    ref = GD.histogram_from_outputs(c["expected"], c["idx"], c["ks"], c["hist_k"])
    for k in ("keys", "det", "steric", "rep_det", "rep_any", "tallies"):
        assert np.array_equal(getattr(h, k).astype(np.int64), ref[k].astype(np.int64)), k
    assert h.total == c["idx"].shape[0]


def test_checkpoint_roundtrip(tmp_path):
    c, h = _hist()
    p = os.path.join(tmp_path, "h.ckpt")
    h.save(p, extra=dict(chunks_done=3))
    h2, extra = C.Histogram.load(p)
    assert h2 == h and extra["chunks_done"] == 3
    with open(p, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(ValueError):
        C.Histogram.load(p)


def test_csv_schema():
    c, h = _hist()
    txt = h.to_csv(space=G.SearchSpace(2, 8))
    lines = txt.strip().split("\n")
    assert lines[0] == "hash_hex,width,height,cell_count,det_count,steric_count,representative_genome,frequency"
    assert len(lines) == len(h) + 1
    f = lines[1].split(",")
    assert f[0].startswith("0x") and len(f[0]) == 10 and f[6].endswith("/24")
    s = h.summary()
    assert s["distinct_hashes"] == len(h)
