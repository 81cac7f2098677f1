"""GPU: the reference-facing Python APIs (assembly.*, classify.enumerate_space with
checkpoint/resume, CSV) on top of the CUDA path, checked against the oracle."""
import os

import numpy as np
import pytest

from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch
    assert torch.cuda.is_available()
    from paper_2205_15311_b200 import assembly, classify, genome
    return assembly, classify, genome


def _edges(tiles):
    from paper_2205_15311_b200._kernels import edges_from_labels
    return edges_from_labels(np.array([v for t in tiles for v in t], np.uint8), len(tiles))


def test_assemble_once_and_classify_tileset(mods):
    from oracle import oracle as O
    A, C, Gm = mods
    rng = np.random.default_rng(5)
    for _ in range(60):
        a = int(rng.integers(1, 4))
        ts = Gm.TileSet(tuple(tuple(int(x) for x in rng.integers(0, 8, 4)) for _ in range(a)))
        out = A.assemble_once(ts, 19, seed=3, genome_index=11, run_index=2)
        grid = np.empty(361, np.int16)
        res = O.assemble_single(_edges(ts.tiles), a, 19, 3, 11, 2, True, grid)
        kind = {0: A.OutcomeKind.BOUNDED, 1: A.OutcomeKind.TRIVIAL_NONDET, 2: A.OutcomeKind.UNBOUND}[res[0]]
        assert out.kind is kind
        if kind is A.OutcomeKind.BOUNDED:
            assert np.array_equal(out.grid.cells.reshape(-1), grid)
        cl = A.classify_tileset(ts, 19, k=8, seed=3, genome_index=11)
        sw = np.zeros(6, np.uint64)
        st, cls, hs, w, h, nc = O.classify_single(_edges(ts.tiles), a, 19, 8, 3, 11, True, sw)
        assert cl.kind.value == ["deterministic", "trivial_nondet", "steric_nondet", "unbound"][cls]
        if cls == 0:
            assert cl.shape_hash == hs and C.shape_hash(cl.shape) == hs
            assert cl.shape == C.CroppedShape.from_packed_words(w, h, sw)


def test_rotation_invariant_classification(mods):
    A, C, Gm = mods
    ts = Gm.TileSet(((2, 0, 0, 0), (0, 0, 1, 0)))      # vertical dimer: deterministic
    a = A.classify_tileset(ts, rotation_invariant=True)
    b = A.classify_tileset(ts)
    assert a.kind is A.ClassKind.DETERMINISTIC and b.kind is A.ClassKind.DETERMINISTIC
    assert a.shape_hash == C.rotation_invariant_hash(b.shape)
    assert A.classify_tileset(Gm.TileSet(((2, 0, 1, 0), (0, 0, 0, 0))), rotation_invariant=True).kind \
        is A.ClassKind.UNBOUND


def test_checkpoint_resume_equals_uninterrupted(mods, tmp_path):
    A, C, Gm = mods
    sp = Gm.SearchSpace(2, 8)
    ck = os.path.join(tmp_path, "enum.ckpt")
    full = C.enumerate_space(sp, ks=(1, 2, 4, 8), start=0x800000, count=1 << 20, batch_size=1 << 17)
    # interrupt the run during batch 4 of 8 (the checkpoint written after batch 3 survives)
    class Stop(Exception):
        pass

    def stop_at_4(done, total):
        if done == 4:
            raise Stop

    with pytest.raises(Stop):
        C.enumerate_space(sp, ks=(1, 2, 4, 8), start=0x800000, count=1 << 20, batch_size=1 << 17, checkpoint=ck,
                          checkpoint_every=1, progress=stop_at_4)
    _, extra = C.Histogram.load(ck)
    assert extra["chunks_done"] == 3 and extra["chunks_total"] == 8
    resumed = C.enumerate_space(sp, ks=(1, 2, 4, 8), start=0x800000, count=1 << 20, batch_size=1 << 17, resume=ck)
    assert resumed == full
    # a checkpoint only resumes the very same plan and space (no silent double counting)
    for kw in (dict(batch_size=1 << 16), dict(count=1 << 19), dict(start=0x800000 + (1 << 17))):
        args = dict(ks=(1, 2, 4, 8), start=0x800000, count=1 << 20, batch_size=1 << 17, resume=ck)
        args.update(kw)
        with pytest.raises(ValueError):
            C.enumerate_space(sp, **args)
    with pytest.raises(ValueError):
        C.enumerate_space(sp, ks=(1, 2, 4, 8), seed=1, start=0x800000, count=1 << 20, batch_size=1 << 17, resume=ck)
    with pytest.raises(ValueError):  # same a, b, d, seed: only the fixed mask differs
        C.enumerate_space(Gm.SearchSpace(2, 8, ((0, 0),)), ks=(1, 2, 4, 8), start=0, count=1 << 20,
                          batch_size=1 << 17, resume=ck)
    with pytest.raises(ValueError):  # indices past the end of the space would alias
        C.enumerate_space(sp, ks=(8,), start=(1 << 24) - 10, count=20)
    hg = G.hist_golden("s28_1m")
    assert np.array_equal(full.keys, hg["keys"]) and np.array_equal(full.tallies, hg["tallies"])
    txt = full.to_csv()
    assert txt.count("\n") == len(full) + 1


def test_enumerate_s32_inert2_building_blocks(mods):
    """SPEC ACCEPTANCE 6 substitute: every deterministic shape of the tile-2-inert S32 slice is a S28 shape."""
    A, C, Gm = mods
    s28 = C.enumerate_space(Gm.SearchSpace(2, 8), ks=(1, 2, 4, 8), batch_size=1 << 24)
    shapes28 = set(s28.keys.tolist())  # DET or steric-attributed shapes of S_{2,8}
    sp = Gm.space_from_preset("s32_3_8_inert2")
    h = C.enumerate_space(sp, ks=(7,), batch_size=1 << 20)
    assert h.total == sp.cardinality
    det = set(h.keys[h.det > 0].tolist())
    assert det and det <= shapes28
