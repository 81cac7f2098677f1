"""JaTAM assembly and k-run classification entry points.

API-compatible with ``tilevolve.assembly`` (/root/reference/pkg/src/tilevolve/
assembly.py, cited "asm:LINE"): every public name keeps its meaning, but the
work runs on the GPU through ``_kernels.assemble_single`` (one movelist run)
and ``_kernels.classify_single`` (k-run fold).  The reference's
``classify_tileset`` cannot run as shipped (it imports the absent
``tilevolve.classify``, asm:197); here it is backed by ``.classify``.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _kernels
from .genome import TileSet

DEFAULT_GRID_DIM = 19  # 19x19 boards (asm:24)


class AssemblyError(ValueError):
    """Bad assembly arguments such as an even grid dimension (asm:27-28)."""


def _partner(label: int) -> int:
    """The label that bonds ``label``: 1<->2, 3<->4, ...; 0 has none."""
    return 0 if label <= 0 else (((label - 1) ^ 1) + 1)


def bonds(i: int, j: int) -> bool:
    """Pair-bonding matrix M_ij (asm:31-33)."""
    return i > 0 and _partner(i) == j


def tile_edges_in_situ(tile, orientation: int) -> tuple[int, int, int, int]:
    """Edge labels facing N, E, S, W after a clockwise quarter-turn x orientation."""
    r = orientation & 3
    return (tile[-r & 3], tile[(1 - r) & 3], tile[(2 - r) & 3], tile[(3 - r) & 3])


@dataclass(frozen=True)
class BondingTable:
    """label -> ((tile, orientation), ...) whose north edge bonds that label,
    one entry per distinct in-situ configuration of a tile (asm:40-58)."""

    entries: tuple[tuple[tuple[int, int], ...], ...]

    def __getitem__(self, label: int) -> tuple[tuple[int, int], ...]:
        return self.entries[label]

    def entries_for(self, label: int, facing: int = 0) -> tuple[tuple[int, int], ...]:
        """The same placements turned so the bonding edge faces ``facing``."""
        return tuple((tile, (rot + facing) % 4) for tile, rot in self.entries[label])


def build_bonding_table(t: TileSet, b: int) -> BondingTable:
    """Bonding-table preprocessing of the movelist algorithm."""
    per_label = [[] for _ in range(b)]
    for ti, tile in enumerate(t.tiles):
        configs = {}
        for rot in range(4):
            configs.setdefault(tile_edges_in_situ(tile, rot), rot)
        for situ, rot in sorted(configs.items(), key=lambda kv: kv[1]):
            owner = _partner(situ[0])
            if 0 < owner < b and situ[0] > 0:
                per_label[owner].append((ti, rot))
    return BondingTable(tuple(tuple(v) for v in per_label))


class OutcomeKind(Enum):
    """Result of one run."""
    BOUNDED = "bounded"
    UNBOUND = "unbound"
    TRIVIAL_NONDET = "trivial_nondet"


class ClassKind(Enum):
    """Result of k runs."""
    DETERMINISTIC = "deterministic"
    TRIVIAL_NONDET = "trivial_nondet"
    STERIC_NONDET = "steric_nondet"
    UNBOUND = "unbound"


_KIND_OF_CODE = dict(zip((_kernels.CLS_DETERMINISTIC, _kernels.CLS_TRIVIAL, _kernels.CLS_STERIC,
                          _kernels.CLS_UNBOUND), ClassKind))
_RUN_OF_CODE = {_kernels.RUN_BOUNDED: OutcomeKind.BOUNDED, _kernels.RUN_UNBOUND: OutcomeKind.UNBOUND,
                _kernels.RUN_TRIVIAL: OutcomeKind.TRIVIAL_NONDET}


class AssemblyGrid:
    """d x d board of int16 cells: -1 empty, else tile*4 + orientation."""

    __slots__ = ("d", "cells")

    def __init__(self, d: int, cells: np.ndarray | None = None):
        self.d = d
        self.cells = (np.full(d * d, -1, np.int16) if cells is None else cells).reshape(d, d)

    def cell(self, row: int, col: int):
        """(tile, orientation) at a cell, or None."""
        v = int(self.cells[row, col])
        return divmod(v, 4) if v >= 0 else None

    def occupancy(self) -> np.ndarray:
        return self.cells >= 0

    def occupied_count(self) -> int:
        return int(np.count_nonzero(self.cells >= 0))

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, AssemblyGrid):
            return False
        return other.d == self.d and np.array_equal(other.cells, self.cells)


@dataclass(frozen=True)
class AssemblyOutcome:
    kind: OutcomeKind
    grid: AssemblyGrid | None = None  # only for BOUNDED


@dataclass(frozen=True)
class Classification:
    kind: ClassKind
    shape_hash: int | None = None  # only for DETERMINISTIC
    shape: "object | None" = None  # CroppedShape, only for DETERMINISTIC


def _check_dim(d: int) -> None:
    if d % 2 == 0 or d < 3:
        raise AssemblyError(f"grid dimension must be odd and >= 3, got {d}")


def _edges_array(t: TileSet) -> tuple[np.ndarray, int]:
    flat = [v for tile in t.tiles for v in tile]
    bad = [v for v in flat if not 0 <= v < 256]
    if bad:
        raise AssemblyError(f"edge label {bad[0]} out of byte range")
    return _kernels.edges_from_labels(np.array(flat, np.uint8), len(t)), len(t)


def assemble_once(t: TileSet, d: int = DEFAULT_GRID_DIM, seed: int = 0, genome_index: int = 0,
                  run_index: int = 0, strict_contacts: bool = True) -> AssemblyOutcome:
    """One movelist run on the device, substream (seed, genome_index, run_index)."""
    _check_dim(d)
    edges, a = _edges_array(t)
    board = np.empty(d * d, np.int16)
    code = _kernels.assemble_single(edges, a, d, np.uint64(seed), np.uint64(genome_index), run_index,
                                    strict_contacts, board)[0]
    if code not in _RUN_OF_CODE:
        raise RuntimeError("movelist capacity exceeded (internal error)")
    kind = _RUN_OF_CODE[code]
    return AssemblyOutcome(kind, AssemblyGrid(d, board) if kind is OutcomeKind.BOUNDED else None)


def _classify_rotation_invariant(t, d, k, seed, genome_index, strict_contacts) -> Classification:
    from .classify import crop, shape_labels

    outcomes = []
    for run in range(k):
        o = assemble_once(t, d, seed=seed, genome_index=genome_index, run_index=run,
                          strict_contacts=strict_contacts)
        if o.kind is OutcomeKind.TRIVIAL_NONDET:
            return Classification(ClassKind.TRIVIAL_NONDET)
        outcomes.append(o)
    if any(o.kind is OutcomeKind.UNBOUND for o in outcomes):
        return Classification(ClassKind.UNBOUND)
    shapes = [crop(o.grid) for o in outcomes]
    W = max(1, (max(s.width * s.height for s in shapes) + 63) // 64)
    rot4, _ = shape_labels([s.width for s in shapes], [s.height for s in shapes],
                           np.stack([s.packed_words(W) for s in shapes]))
    labels = {int(v) for v in rot4}
    if len(labels) > 1:
        return Classification(ClassKind.STERIC_NONDET)
    return Classification(ClassKind.DETERMINISTIC, labels.pop(), shapes[0])


def classify_tileset(t: TileSet, d: int = DEFAULT_GRID_DIM, k: int = 8, seed: int = 0, genome_index: int = 0,
                     strict_contacts: bool = True, rotation_invariant: bool = False) -> Classification:
    """k-redundant classification with precedence TRIVIAL > UNBOUND > STERIC
    (SPEC.md:174-182, 318).  ``rotation_invariant`` compares the sorted-four-
    rotation hashes instead of plain shape hashes."""
    _check_dim(d)
    if k < 1:
        raise AssemblyError(f"redundancy k must be >= 1, got {k}")
    if rotation_invariant:
        return _classify_rotation_invariant(t, d, k, seed, genome_index, strict_contacts)
    from .classify import CroppedShape

    edges, a = _edges_array(t)
    words = np.zeros((d * d + 63) // 64, np.uint64)
    status, code, hsh, w, h, _ = _kernels.classify_single(edges, a, d, k, np.uint64(seed), np.uint64(genome_index),
                                                          strict_contacts, words)
    if status:
        raise RuntimeError("movelist capacity exceeded (internal error)")
    kind = _KIND_OF_CODE[code]
    if kind is ClassKind.DETERMINISTIC:
        return Classification(kind, int(hsh), CroppedShape.from_packed_words(int(w), int(h), words))
    return Classification(kind)


def outcome_equivalent(a: AssemblyGrid, b: AssemblyGrid) -> bool:
    """Position-sensitive configuration equivalence."""
    if a.d != b.d:
        raise AssemblyError(f"grid dimensions differ: {a.d} vs {b.d}")
    return a == b
