"""GPU: canonical shape labels (tv_shape_labels) -- the SPEC.md:270-278
rotation-invariant hash and the D4 min-hash -- against the host definitions
in classify.py, on every record of the full-S_{2,8} reference histogram and
on random shapes, plus group invariance."""
import numpy as np
import pytest

from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def C():
    import torch
    assert torch.cuda.is_available()
    from paper_2205_15311_b200 import classify
    return classify


def _host_labels(C, w, h, shape):
    rot4, d4 = [], []
    for i in range(len(w)):
        s = C.CroppedShape.from_packed_words(int(w[i]), int(h[i]), shape[i])
        rot4.append(C.rotation_invariant_hash(s))
        d4.append(C.d4_min_hash(s))
    return np.array(rot4, np.uint32), np.array(d4, np.uint32)


def test_labels_on_reference_histogram(C):
    z = G.hist_golden("s28_full")
    rot4, d4 = C.shape_labels(z["w"], z["h"], z["shape"])
    hr, hd = _host_labels(C, z["w"], z["h"], z["shape"])
    assert np.array_equal(rot4, hr)
    assert np.array_equal(d4, hd)
    # the plain hash is one of the 8 transforms, so d4 <= key
    assert np.all(d4 <= z["keys"])


def test_labels_random_shapes_and_invariance(C):
    rng = np.random.default_rng(11)
    shapes = []
    for _ in range(400):
        w, h = int(rng.integers(1, 18)), int(rng.integers(1, 18))
        b = rng.random((h, w)) < rng.uniform(0.2, 0.9)
        b[0, rng.integers(0, w)] = True  # keep the crop tight on at least the first row
        shapes.append(C.CroppedShape(w, h, b))
    W = 5
    for variant in range(8):
        vs = [s.rotated(variant & 3) if variant < 4 else s.mirrored().rotated(variant & 3) for s in shapes]
        w = np.array([s.width for s in vs], np.uint8)
        h = np.array([s.height for s in vs], np.uint8)
        sh = np.stack([s.packed_words(W) for s in vs])
        rot4, d4 = C.shape_labels(w, h, sh)
        if variant == 0:
            hr, hd = _host_labels(C, w, h, sh)
            assert np.array_equal(rot4, hr) and np.array_equal(d4, hd)
            base_r, base_d = rot4, d4
        assert np.array_equal(d4, base_d)          # D4-invariant
        if variant < 4:
            assert np.array_equal(rot4, base_r)    # rotation-invariant


def test_canonical_classes_fold(C):
    z = G.hist_golden("s28_full")
    H = C.Histogram((1, 2, 4, 8), 8, 6, keys=z["keys"], det=z["det"], steric=z["steric"], rep_det=z["rep_det"],
                    rep_any=z["rep_any"], w=z["w"], h=z["h"], cells=z["cells"], shape=z["shape"],
                    tallies=z["tallies"])
    for kind in ("d4", "rot4"):
        cc = H.canonical_classes(kind)
        assert int(cc["det"].sum()) == int(z["det"].sum())
        assert int(cc["steric"].sum()) == int(z["steric"].sum())
        assert int(cc["hashes"].sum()) == len(z["keys"])
        assert np.all(np.diff(cc["label"].astype(np.int64)) > 0)
    assert len(H.canonical_classes("d4")["label"]) <= len(H.canonical_classes("rot4")["label"])


def test_empty_and_oversized_rows(C):
    rot4, d4 = C.shape_labels(np.zeros(0, np.uint8), np.zeros(0, np.uint8), np.zeros((0, 2), np.uint64))
    assert rot4.shape == (0,)
    # 9x9 = 81 bits do not fit W = 1 word -> label 0
    rot4, d4 = C.shape_labels(np.array([9, 2], np.uint8), np.array([9, 2], np.uint8),
                              np.array([[~np.uint64(0)], [np.uint64(15)]], np.uint64))
    assert rot4[0] == 0 and d4[0] == 0 and rot4[1] != 0


def test_labels_large_shapes(C):
    """Crops of large grids (up to 120 x 120, W = 225 words) against the host definitions,
    D4 invariance included."""
    rng = np.random.default_rng(29)
    shapes = []
    for _ in range(40):
        w, h = int(rng.integers(1, 121)), int(rng.integers(1, 121))
        b = rng.random((h, w)) < rng.uniform(0.05, 0.6)
        b[0, rng.integers(0, w)] = True
        b[rng.integers(0, h), 0] = True
        shapes.append(C.CroppedShape(w, h, b))
    W = (120 * 120 + 63) // 64
    for variant in (0, 1, 5):
        vs = [s.rotated(variant & 3) if variant < 4 else s.mirrored().rotated(variant & 3) for s in shapes]
        w = np.array([s.width for s in vs], np.uint8)
        h = np.array([s.height for s in vs], np.uint8)
        sh = np.stack([s.packed_words(W) for s in vs])
        rot4, d4 = C.shape_labels(w, h, sh)
        if variant == 0:
            hr, hd = _host_labels(C, w, h, sh)
            assert np.array_equal(rot4, hr) and np.array_equal(d4, hd)
            base_r, base_d = rot4, d4
        assert np.array_equal(d4, base_d)
        if variant < 4:
            assert np.array_equal(rot4, base_r)
