"""Shape extraction, hashing and exhaustive enumeration into a phenotype histogram.

The reference ships no ``tilevolve.classify`` (asm:197 imports it; it is only
specified in SPEC.md:220-327).  This module provides that contract with the
enumeration running on the device: ``enumerate_space`` streams index chunks
through ``tv_enumerate_range`` (fused decode -> k runs -> fold -> on-device
histogram), so no per-genome data ever leaves HBM.  The per-genome parity
anchor is the reference ``classify_batch`` (_k:404-452): the histogram is the
aggregation SPEC.md:235-240/297-306 defines over its outputs.

Histogram columns per shape hash: det_count, steric_count, the lowest DET
enumeration index (rep_det), the lowest DET-or-STERIC index (rep_any,
SPEC.md:300 "representative genome = lowest enumeration index"), width,
height, cell count and the cropped bitmap.  Global tallies per prefix k in
the order DET, TRIV, STERIC, UNB, ERROR.
"""
from __future__ import annotations

import ctypes
import hashlib
import io
import json
import math
import os
import struct
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .genome import SearchSpace, genome_at_index

OAT_MASK = 0xFFFFFFFF


def _oat(data) -> int:
    h = 0
    for k in data:
        h = (h + int(k)) & OAT_MASK
        h = (h + (h << 10)) & OAT_MASK
        h ^= h >> 6
    h = (h + (h << 3)) & OAT_MASK
    h ^= h >> 11
    return (h + (h << 15)) & OAT_MASK


def oat_hash(data) -> int:
    """Jenkins one-at-a-time hash (device twin _k:79-85 /
    tv_oat_hash_bytes).  Host utility for single shapes."""
    return _oat(bytes(np.asarray(data, dtype=np.uint8).reshape(-1)))


@dataclass(frozen=True, eq=False)
class CroppedShape:
    """Tight bounding box of an assembly."""

    width: int
    height: int
    bitmap: np.ndarray  # (height, width) bool, row-major
    origin: tuple[int, int] = (0, 0)  # (row, col) of the box in the source grid

    @property
    def cells(self) -> int:
        return int(self.bitmap.sum())

    @classmethod
    def from_packed_words(cls, w: int, h: int, words) -> "CroppedShape":
        """Inverse of the kernel's packing: bit y*w+x, LSB-first per u64 (_k:280-292)."""
        wd = np.asarray(words, dtype=np.uint64)
        bits = np.unpackbits(wd.view(np.uint8), bitorder="little")[: w * h]
        return cls(int(w), int(h), bits.reshape(h, w).astype(bool))

    def packed_words(self, W: int) -> np.ndarray:
        flat = np.zeros(W * 64, np.uint8)
        flat[: self.width * self.height] = self.bitmap.reshape(-1)
        return np.packbits(flat, bitorder="little").view(np.uint64).copy()

    def rotated(self, quarter_turns: int = 1) -> "CroppedShape":
        """Clockwise rotation by 90 degrees x quarter_turns."""
        b = np.rot90(self.bitmap, -quarter_turns)
        return CroppedShape(b.shape[1], b.shape[0], np.ascontiguousarray(b))

    def mirrored(self) -> "CroppedShape":
        b = np.ascontiguousarray(self.bitmap[:, ::-1])
        return CroppedShape(self.width, self.height, b)

    def __eq__(self, other: object) -> bool:
        return (isinstance(other, CroppedShape) and other.width == self.width and other.height == self.height
                and np.array_equal(other.bitmap, self.bitmap))

    def to_ascii(self) -> str:
        return "\n".join("".join("#" if v else "." for v in row) for row in self.bitmap)


def crop(g) -> CroppedShape:
    """Tight crop of an AssemblyGrid."""
    occ = g.cells >= 0
    rows = np.nonzero(occ.any(axis=1))[0]
    cols = np.nonzero(occ.any(axis=0))[0]
    if rows.size == 0:
        raise ValueError("cannot crop an empty grid")
    r0, r1, c0, c1 = rows[0], rows[-1], cols[0], cols[-1]
    return CroppedShape(int(c1 - c0 + 1), int(r1 - r0 + 1), occ[r0:r1 + 1, c0:c1 + 1].copy(), (int(r0), int(c0)))


def shape_hash(s: CroppedShape) -> int:
    """OAT over width, height, then (x, y) of occupied cells row-major
    (identical to the kernel's _hash_region, _k:260-277)."""
    if s.width > 255 or s.height > 255:
        raise ValueError("shape larger than 255 cells per side")
    ys, xs = np.nonzero(s.bitmap)
    seq = [s.width, s.height]
    for y, x in zip(ys.tolist(), xs.tolist()):
        seq += [x, y]
    return _oat(seq)


def rotation_invariant_hash(s: CroppedShape) -> int:
    """Sorted hashes of the four rotations, re-hashed as 16 little-endian bytes
    (SPEC.md:270-278).  Reflections are not included."""
    hs = sorted(shape_hash(s.rotated(k)) for k in range(4))
    return _oat(struct.pack("<4I", *hs))


def d4_min_hash(s: CroppedShape) -> int:
    """Extra canonical label: minimum shape_hash over the 8 rotations and
    reflections (dihedral group D4).  Not used for classification (the
    reference key is the plain shape_hash)."""
    return min(min(shape_hash(s.rotated(k)), shape_hash(s.mirrored().rotated(k))) for k in range(4))


def shapediff(A, B) -> int:
    """Number of grid positions whose empty/occupied status differs."""
    if A.d != B.d:
        raise ValueError(f"grid dimensions differ: {A.d} vs {B.d}")
    return int(np.count_nonzero(A.occupancy() != B.occupancy()))


def shapesim(A, B) -> float:
    return 1.0 - shapediff(A, B) / float(A.d * A.d)


def collision_probability(n: int) -> float:
    """Birthday bound of Eq. 2 for n distinct phenotypes, 1 - prod_{i<n} (1 - i 2^-32).
    SPEC.md:288-296 writes the upper limit as n but its worked example
    (n=2 -> 2^-32) and the paper's Eq. 2 use i = 0..n-1; the example wins."""
    if n < 0:
        raise ValueError("n must be >= 0")
    i = np.arange(max(n, 0), dtype=np.float64)
    return float(-np.expm1(np.sum(np.log1p(-i * 2.0 ** -32))))


# --------------------------------------------------------------------------- histogram

_CKPT_MAGIC = b"TVHIST\x00\x01"
_CKPT_VERSION = 1
CLASS_NAMES = ("DET", "TRIV", "STERIC", "UNB", "ERROR")


@dataclass(eq=False)
class Histogram:
    """Merged per-shape-hash records plus per-k class tallies."""

    ks: tuple
    hist_k: int
    W: int
    keys: np.ndarray = None       # u32, ascending
    det: np.ndarray = None        # u64
    steric: np.ndarray = None     # u64
    rep_det: np.ndarray = None    # u64, UINT64_MAX = none
    rep_any: np.ndarray = None    # u64
    w: np.ndarray = None          # u8
    h: np.ndarray = None          # u8
    cells: np.ndarray = None      # u16
    shape: np.ndarray = None      # u64 [U, W]
    tallies: np.ndarray = None    # i64 [q, 5]
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.keys is None:
            self.keys = np.zeros(0, np.uint32)
            for n, dt in (("det", np.uint64), ("steric", np.uint64), ("rep_det", np.uint64), ("rep_any", np.uint64),
                          ("w", np.uint8), ("h", np.uint8), ("cells", np.uint16)):
                setattr(self, n, np.zeros(0, dt))
            self.shape = np.zeros((0, self.W), np.uint64)
        if self.tallies is None:
            self.tallies = np.zeros((len(self.ks), 5), np.int64)
        self.ks = tuple(int(k) for k in self.ks)

    # -- views
    def __len__(self) -> int:
        return int(self.keys.shape[0])

    @property
    def total(self) -> int:
        """Genomes tallied (every prefix row sums to this)."""
        return int(self.tallies[0].sum())

    def class_counts(self, k: int | None = None) -> dict:
        row = self.tallies[self.ks.index(self.hist_k if k is None else k)]
        return dict(zip(CLASS_NAMES, (int(v) for v in row)))

    def shape_of(self, i: int) -> CroppedShape:
        return CroppedShape.from_packed_words(int(self.w[i]), int(self.h[i]), self.shape[i])

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, Histogram):
            return False
        if self.ks != other.ks or self.hist_k != other.hist_k or self.W != other.W:
            return False
        return all(np.array_equal(getattr(self, n), getattr(other, n))
                   for n in ("keys", "det", "steric", "rep_det", "rep_any", "w", "h", "cells", "shape", "tallies"))

    @classmethod
    def from_rows(cls, indices, out_class, out_hash, out_w, out_h, out_cells, out_shape, ks, hist_k,
                  W: int | None = None, meta: dict | None = None) -> "Histogram":
        """Aggregate per-genome classify_batch rows (_k:404-452) into a Histogram
        (host; used to fold classify_batch results and by the tests)."""
        ks = tuple(int(k) for k in ks)
        W = int(W if W is not None else out_shape.shape[1])
        idx = np.asarray(indices, np.uint64)
        cls_ = np.asarray(out_class)
        out = cls(ks, int(hist_k), W, meta=dict(meta or {}))
        for j in range(len(ks)):
            c = cls_[:, j]
            for v, col in ((0, 0), (1, 1), (2, 2), (3, 3), (255, 4)):
                out.tallies[j, col] = int(np.count_nonzero(c == v))
        hc = cls_[:, ks.index(int(hist_k))]
        sel = np.nonzero((hc == 0) | (hc == 2))[0]
        keys, inv = np.unique(np.asarray(out_hash)[sel], return_inverse=True)
        U = keys.shape[0]
        isdet = hc[sel] == 0
        out.keys = keys.astype(np.uint32)
        out.det = np.bincount(inv, weights=isdet, minlength=U).astype(np.uint64)
        out.steric = np.bincount(inv, weights=~isdet, minlength=U).astype(np.uint64)
        big = np.iinfo(np.uint64).max
        out.rep_det = np.full(U, big, np.uint64)
        out.rep_any = np.full(U, big, np.uint64)
        np.minimum.at(out.rep_any, inv, idx[sel])
        np.minimum.at(out.rep_det, inv[isdet], idx[sel][isdet])
        # payload = the representative's row (lowest index per key), whatever the row order
        order = np.lexsort((idx[sel], inv))
        starts = np.r_[0, np.flatnonzero(np.diff(inv[order])) + 1] if sel.size else np.zeros(0, np.int64)
        rows = sel[order[starts]]
        out.w = np.asarray(out_w)[rows].astype(np.uint8)
        out.h = np.asarray(out_h)[rows].astype(np.uint8)
        out.cells = np.asarray(out_cells)[rows].astype(np.uint16)
        sh = np.zeros((U, W), np.uint64)
        src = np.asarray(out_shape)[rows]
        k = min(W, src.shape[1])
        sh[:, :k] = src[:, :k]
        out.shape = sh
        return out

    # -- merging (host; commutative and associative)
    @staticmethod
    def merge_many(parts: list["Histogram"]) -> "Histogram":
        first = parts[0]
        for p in parts[1:]:
            if p.ks != first.ks or p.hist_k != first.hist_k or p.W != first.W:
                raise ValueError("histograms with different ks / hist_k / W cannot be merged")
        keys = np.concatenate([p.keys for p in parts])
        u, inv = np.unique(keys, return_inverse=True)
        U = u.shape[0]
        out = Histogram(first.ks, first.hist_k, first.W, meta=dict(first.meta))
        out.keys = u.astype(np.uint32)
        det = np.zeros(U, np.uint64)
        ste = np.zeros(U, np.uint64)
        np.add.at(det, inv, np.concatenate([p.det for p in parts]))
        np.add.at(ste, inv, np.concatenate([p.steric for p in parts]))
        out.det, out.steric = det, ste
        for n in ("rep_det", "rep_any"):
            r = np.full(U, np.iinfo(np.uint64).max, np.uint64)
            np.minimum.at(r, inv, np.concatenate([getattr(p, n) for p in parts]))
            setattr(out, n, r)
        # payload of each key = the one travelling with its lowest rep_any (ties: first part)
        ra = np.concatenate([p.rep_any for p in parts])
        order = np.lexsort((np.arange(keys.shape[0]), ra, inv))
        starts = np.r_[0, np.flatnonzero(np.diff(inv[order])) + 1] if keys.shape[0] else np.zeros(0, np.int64)
        first_pos = order[starts]
        for n in ("w", "h", "cells"):
            setattr(out, n, np.concatenate([getattr(p, n) for p in parts])[first_pos])
        out.shape = np.concatenate([p.shape for p in parts])[first_pos].reshape(U, first.W)
        out.tallies = np.sum([p.tallies for p in parts], axis=0).astype(np.int64)
        return out

    def merge(self, other: "Histogram") -> "Histogram":
        return Histogram.merge_many([self, other])

    # -- result formats
    def to_csv(self, path_or_buf=None, cardinality: int | None = None, space: SearchSpace | None = None) -> str:
        """``hash_hex,width,height,cell_count,det_count,steric_count,representative_genome,frequency``
        one row per hash (ascending); frequency = det_count / cardinality."""
        space = space or self._space()
        card = cardinality or (space.cardinality if space else max(1, self.total))
        buf = io.StringIO()
        buf.write("hash_hex,width,height,cell_count,det_count,steric_count,representative_genome,frequency\n")
        for i in range(len(self)):
            rep = int(self.rep_any[i])
            rep_txt = genome_at_index(space, rep).to_text() if space is not None else str(rep)
            buf.write(f"0x{int(self.keys[i]):08x},{int(self.w[i])},{int(self.h[i])},{int(self.cells[i])},"
                      f"{int(self.det[i])},{int(self.steric[i])},{rep_txt},{int(self.det[i]) / card:.12g}\n")
        text = buf.getvalue()
        if path_or_buf is not None:
            if hasattr(path_or_buf, "write"):
                path_or_buf.write(text)
            else:
                with open(path_or_buf, "w") as f:
                    f.write(text)
        return text

    def summary(self) -> dict:
        """Summary JSON: totals per class per k, parameters, runtime."""
        return dict(
            params=self.meta,
            ks=list(self.ks), hist_k=self.hist_k,
            totals={str(k): dict(zip(CLASS_NAMES, (int(v) for v in self.tallies[i]))) for i, k in enumerate(self.ks)},
            distinct_hashes=len(self),
            deterministic_hashes=int(np.count_nonzero(self.det)),
            steric_hashes=int(np.count_nonzero(self.steric)),
        )

    def _space(self):
        m = self.meta
        if "a" in m and "b" in m:
            return SearchSpace(m["a"], m["b"], tuple(tuple(x) for x in m.get("fixed_mask", ())))
        return None

    # -- canonical phenotype classes (extra columns; the key stays the plain hash)
    def canonical_labels(self, stream=None) -> dict:
        """Per-record canonical labels computed on the device (tv_shape_labels):
        ``rot4`` = SPEC.md:270-278 rotation-invariant hash, ``d4`` = minimum
        shape hash over the 8 rotations and reflections."""
        rot4, d4 = shape_labels(self.w, self.h, self.shape, stream=stream)
        return dict(rot4=rot4, d4=d4)

    def canonical_classes(self, kind: str = "d4", stream=None) -> dict:
        """Records folded by canonical label: per label the summed det / steric
        counts, the lowest representatives and how many plain hashes map to it.
        Sorted by label."""
        if kind not in ("d4", "rot4"):
            raise ValueError("kind must be 'd4' or 'rot4'")
        lab = self.canonical_labels(stream)[kind]
        u, inv = np.unique(lab, return_inverse=True)
        U = u.shape[0]
        det = np.zeros(U, np.uint64)
        ste = np.zeros(U, np.uint64)
        np.add.at(det, inv, self.det)
        np.add.at(ste, inv, self.steric)
        big = np.iinfo(np.uint64).max
        rep_det = np.full(U, big, np.uint64)
        rep_any = np.full(U, big, np.uint64)
        np.minimum.at(rep_det, inv, self.rep_det)
        np.minimum.at(rep_any, inv, self.rep_any)
        return dict(label=u.astype(np.uint32), det=det, steric=ste, rep_det=rep_det, rep_any=rep_any,
                    hashes=np.bincount(inv, minlength=U).astype(np.int64))

    # -- checkpoint: versioned binary layout
    #   magic 8B | version u32 | header_len u32 | header JSON (utf-8) | arrays in header["arrays"] order, raw LE
    def save(self, path: str, extra: dict | None = None) -> None:
        arrays = ("keys", "det", "steric", "rep_det", "rep_any", "w", "h", "cells", "shape", "tallies")
        header = dict(ks=list(self.ks), hist_k=self.hist_k, W=self.W, n=len(self), meta=self.meta,
                      extra=extra or {}, arrays=[[a, str(getattr(self, a).dtype), list(getattr(self, a).shape)]
                                                 for a in arrays])
        hb = json.dumps(header).encode()
        tmp = path + ".tmp"
        with open(tmp, "wb") as f:
            f.write(_CKPT_MAGIC)
            f.write(struct.pack("<II", _CKPT_VERSION, len(hb)))
            f.write(hb)
            for a in arrays:
                f.write(np.ascontiguousarray(getattr(self, a)).tobytes())
        os.replace(tmp, path)

    @classmethod
    def load(cls, path: str) -> tuple["Histogram", dict]:
        with open(path, "rb") as f:
            if f.read(8) != _CKPT_MAGIC:
                raise ValueError(f"{path}: not a tilevolve histogram checkpoint")
            ver, hl = struct.unpack("<II", f.read(8))
            if ver != _CKPT_VERSION:
                raise ValueError(f"{path}: checkpoint version {ver} unsupported")
            header = json.loads(f.read(hl))
            out = cls(tuple(header["ks"]), header["hist_k"], header["W"], meta=header["meta"])
            for name, dt, shp in header["arrays"]:
                cnt = int(np.prod(shp)) if shp else 1
                arr = np.frombuffer(f.read(cnt * np.dtype(dt).itemsize), dtype=dt).reshape(shp).copy()
                setattr(out, name, arr)
        return out, header["extra"]


def shape_labels(w, h, shape, stream=None) -> tuple[np.ndarray, np.ndarray]:
    """(rot4, d4) labels of packed cropped shapes on the device (tv_shape_labels).
    ``shape`` is u64[n, W] (bit y*w+x, _k:280-292), ``w``/``h`` u8[n]."""
    w = np.ascontiguousarray(w, np.uint8)
    h = np.ascontiguousarray(h, np.uint8)
    sh = np.ascontiguousarray(shape, np.uint64)
    n = w.shape[0]
    if sh.ndim != 2 or sh.shape[0] != n or h.shape[0] != n:
        raise ValueError("shape must be [n, W] with n = len(w) = len(h)")
    rot4 = np.zeros(n, np.uint32)
    d4 = np.zeros(n, np.uint32)
    P = _lib.ptr
    _lib.check(_lib.lib().tv_shape_labels(P(sh), P(w), P(h), n, max(1, sh.shape[1]), P(rot4), P(d4), stream))
    return rot4, d4


class DeviceHistogram:
    """Device-resident histogram handle (tv_hist_*); one CUDA device."""

    def __init__(self, ks, hist_k: int, W: int, capacity: int = 1 << 20):
        self.ks = tuple(int(k) for k in ks)
        self.hist_k = int(hist_k)
        self.W = int(W)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().tv_hist_create(int(capacity), len(self.ks), self.W, ctypes.byref(h)))
        self._h = h

    def close(self):
        if self._h:
            _lib.lib().tv_hist_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def clear(self, stream=None):
        _lib.check(_lib.lib().tv_hist_clear(self._h, stream))

    def count(self, stream=None) -> tuple[int, bool]:
        n = ctypes.c_int64()
        o = ctypes.c_int32()
        _lib.check(_lib.lib().tv_hist_count(self._h, ctypes.byref(n), ctypes.byref(o), stream))
        return n.value, bool(o.value)

    def enumerate_range(self, space: SearchSpace, start: int, count: int, d: int, seed: int, strict: bool,
                        stream=None) -> None:
        a, bpl, mp, mv, fp = space.kernel_args()
        ks = np.array(self.ks, np.int64)
        _lib.check(_lib.lib().tv_enumerate_range(
            int(start), int(count), a, bpl, _lib.ptr(mp), _lib.ptr(mv), mp.shape[0], _lib.ptr(fp), fp.shape[0],
            int(d), _lib.ptr(ks), ks.shape[0], self.hist_k, int(np.uint64(seed)), int(bool(strict)), self._h, stream))

    def enumerate_chunks(self, space: SearchSpace, start: int, count: int, chunk: int, stride: int, d: int, seed: int,
                         strict: bool, stream=None) -> None:
        """``count`` items in chunks of ``chunk`` consecutive indices, chunk c starting at
        start + c * stride: one launch for a rank's round-robin share (tv_enumerate_chunks)."""
        a, bpl, mp, mv, fp = space.kernel_args()
        ks = np.array(self.ks, np.int64)
        _lib.check(_lib.lib().tv_enumerate_chunks(
            int(start), int(count), int(chunk), int(stride), a, bpl, _lib.ptr(mp), _lib.ptr(mv), mp.shape[0],
            _lib.ptr(fp), fp.shape[0], int(d), _lib.ptr(ks), ks.shape[0], self.hist_k, int(np.uint64(seed)),
            int(bool(strict)), self._h, stream))

    def enumerate_indices(self, space: SearchSpace, indices, d: int, seed: int, strict: bool, stream=None) -> None:
        a, bpl, mp, mv, fp = space.kernel_args()
        ks = np.array(self.ks, np.int64)
        idx = indices if _lib.is_cuda(indices) else np.ascontiguousarray(indices, np.uint64)
        _lib.check(_lib.lib().tv_enumerate_indices(
            _lib.ptr(idx), int(idx.shape[0]), a, bpl, _lib.ptr(mp), _lib.ptr(mv), mp.shape[0], _lib.ptr(fp),
            fp.shape[0], int(d), _lib.ptr(ks), ks.shape[0], self.hist_k, int(np.uint64(seed)), int(bool(strict)),
            self._h, stream or _lib.stream_of(idx)))

    def export(self, stream=None, meta: dict | None = None) -> Histogram:
        n, ovf = self.count(stream)
        if ovf:
            raise _lib.TvError("device histogram overflowed; raise capacity")
        out = Histogram(self.ks, self.hist_k, self.W, meta=dict(meta or {}))
        out.keys = np.zeros(n, np.uint32)
        for name, dt in (("det", np.uint64), ("steric", np.uint64), ("rep_det", np.uint64), ("rep_any", np.uint64),
                         ("w", np.uint8), ("h", np.uint8), ("cells", np.uint16)):
            setattr(out, name, np.zeros(n, dt))
        out.shape = np.zeros((n, self.W), np.uint64)
        out.tallies = np.zeros((len(self.ks), 5), np.int64)
        got = ctypes.c_int64()
        P = _lib.ptr
        _lib.check(_lib.lib().tv_hist_export(self._h, n, P(out.keys), P(out.det), P(out.steric), P(out.rep_det),
                                             P(out.rep_any), P(out.w), P(out.h), P(out.cells), P(out.shape),
                                             P(out.tallies), ctypes.byref(got), stream))
        return out

    @property
    def row_width(self) -> int:
        return 7 + self.W

    def pack_into(self, rows, tallies, stream=None) -> int:
        """Raw records into ``rows`` (torch int64 [>= n, 7 + W], device or host) and the
        tallies into ``tallies`` ([q, 5] int64); returns n (tv_hist_pack)."""
        n = ctypes.c_int64()
        _lib.check(_lib.lib().tv_hist_pack(self._h, int(rows.shape[0]), _lib.ptr(rows), _lib.ptr(tallies),
                                           ctypes.byref(n), stream or _lib.stream_of(rows)))
        return n.value

    def replace_rows(self, rows, tallies, stream=None) -> None:
        """Clear and merge packed rows of several histograms (tv_hist_replace_rows); rows whose
        first word is 0 are padding."""
        _lib.check(_lib.lib().tv_hist_replace_rows(self._h, int(rows.shape[0]), _lib.ptr(rows), _lib.ptr(tallies),
                                                   stream or _lib.stream_of(rows)))

    def merge(self, hist: Histogram, stream=None) -> None:
        P = _lib.ptr
        tal = np.ascontiguousarray(hist.tallies, np.int64)
        _lib.check(_lib.lib().tv_hist_merge(self._h, len(hist), P(hist.keys), P(hist.det), P(hist.steric),
                                            P(hist.rep_det), P(hist.rep_any), P(hist.w), P(hist.h), P(hist.cells),
                                            P(np.ascontiguousarray(hist.shape)), P(tal), stream))


_tls = threading.local()


def _cached_histogram(ks, hist_k, W, capacity) -> "DeviceHistogram":
    """Per-thread reusable device histogram (allocation and its implicit device
    synchronisation stay out of repeated enumerate_space calls); cleared on reuse."""
    import torch
    key = (torch.cuda.current_device() if torch.cuda.is_available() else -1, tuple(ks), int(hist_k), int(W),
           int(capacity))
    cache = getattr(_tls, "hists", None)
    if cache is None:
        cache = _tls.hists = {}
    h = cache.get(key)
    if h is None or h._h is None:
        h = cache[key] = DeviceHistogram(ks, hist_k, W, capacity)
    else:
        h.clear()
    return h


def _drop_cached_histogram(h) -> None:
    cache = getattr(_tls, "hists", {})
    for k, v in list(cache.items()):
        if v is h:
            del cache[k]
    h.close()


def shape_words_for(d: int) -> int:
    """u64 words for the largest bounded crop, (d-2) x (d-2) bits."""
    return max(1, ((d - 2) * (d - 2) + 63) // 64)


def _space_meta(space: SearchSpace, d, seed, strict) -> dict:
    return dict(a=space.a, b=space.b, fixed_mask=[list(x) for x in space.fixed_mask], d=int(d), seed=int(seed),
                strict=bool(strict), cardinality=space.cardinality)


def chunk_plan(start: int, count: int, batch_size: int) -> list[tuple[int, int]]:
    """[start, start+count) cut into batch_size chunks (the enumeration work units)."""
    return [(s, min(batch_size, start + count - s)) for s in range(start, start + count, batch_size)]


def enumerate_space(space: SearchSpace, d: int = 19, k: int = 8, seed: int = 0, batch_size: int = 1 << 26,
                    workers: int | None = None, *, ks=None, hist_k: int | None = None, strict: bool = True,
                    start: int = 0, count: int | None = None, capacity: int = 1 << 20,
                    checkpoint: str | None = None, checkpoint_every: int = 64, resume: str | None = None,
                    progress=None, chunks: list | None = None) -> Histogram:
    """Exhaustively classify [start, start+count) of ``space`` into a Histogram
    (SPEC.md:297-306).  Results are bit-identical for any batch_size (each
    genome's substream depends only on (seed, index, run), _k:45-48).

    ``ks`` (default ``(k,)``) lists the prefix redundancies tallied; the hash
    attribution uses ``hist_k`` (default ``max(ks)``).  ``workers`` is accepted
    for API compatibility; the device kernel schedules genomes itself.
    Checkpoints (versioned binary, every ``checkpoint_every`` batches) store the
    merged records and the chunk cursor; ``resume`` continues from one.
    """
    ks = tuple(sorted(int(x) for x in (ks if ks is not None else (k,))))
    hist_k = int(hist_k if hist_k is not None else ks[-1])
    if count is None:
        count = space.cardinality - start
    if start < 0 or count < 0 or start + count > space.cardinality:
        raise ValueError(f"[start, start+count) = [{start}, {start + count}) is outside the space "
                         f"(cardinality {space.cardinality})")
    W = shape_words_for(d)
    plan = chunks if chunks is not None else chunk_plan(start, count, batch_size)
    for s_, n_ in plan:
        if s_ < 0 or n_ < 0 or s_ + n_ > space.cardinality:
            raise ValueError(f"chunk ({s_}, {n_}) is outside the space (cardinality {space.cardinality})")
    meta = _space_meta(space, d, seed, strict)
    # the chunk cursor of a checkpoint only means something for the very same plan
    cursor = dict(start=int(start), count=int(count), batch_size=int(batch_size), chunks_total=len(plan),
                  plan_sha256=hashlib.sha256(json.dumps([[int(a), int(b)] for a, b in plan]).encode()).hexdigest())
    dev = _cached_histogram(ks, hist_k, W, capacity)
    done = 0
    if resume:
        prev, extra = Histogram.load(resume)
        if prev.ks != ks or prev.hist_k != hist_k or prev.W != W:
            raise ValueError("checkpoint was written with different ks / hist_k / d")
        for key in ("a", "b", "fixed_mask", "d", "seed", "strict"):
            if prev.meta.get(key) != meta[key]:
                raise ValueError(f"checkpoint parameter {key} differs")
        for key, v in cursor.items():
            if extra.get(key) != v:
                raise ValueError(f"checkpoint was written for another chunk plan ({key}: {extra.get(key)!r} "
                                 f"!= {v!r})")
        done = int(extra["chunks_done"])
        if not 0 <= done <= len(plan):
            raise ValueError(f"checkpoint cursor {done} outside the plan of {len(plan)} chunks")
        dev.merge(prev)
    t0 = time.time()
    try:
        for ci in range(done, len(plan)):
            s, n = plan[ci]
            dev.enumerate_range(space, s, n, d, seed, strict)
            if progress is not None:
                progress(ci + 1, len(plan))
            if checkpoint and ((ci + 1) % checkpoint_every == 0 or ci + 1 == len(plan)):
                dev.export(meta=meta).save(checkpoint, extra=dict(cursor, chunks_done=ci + 1))
        out = dev.export(meta=meta)
    except BaseException:
        _drop_cached_histogram(dev)
        raise
    out.meta["runtime_s"] = time.time() - t0
    out.meta["start"] = int(start)
    out.meta["count"] = int(count)
    return out
