"""ctypes view of the CPU restatement (oracle/tv_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's CPU-baseline leg as the checker.  The product package never imports
this module.  Parity status: pinned against golden vectors generated from the
reference (tests/golden/make_golden.py) and SURVEY.md Appendix C digests.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtv_oracle.so")
_lib = None

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_u64 = ctypes.c_uint64


def build() -> str:
    """Compile the restatement with the committed Makefile (gcc, OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_oat_hash_bytes.restype = ctypes.c_uint32
        L.orc_oat_hash_bytes.argtypes = [_p, _i64]
        L.orc_classify_batch.restype = _i32
        L.orc_classify_batch.argtypes = [_p, _i64, _i32, _i32, _p, _p, _i64, _p, _i64, _i32,
                                         _p, _i64, _i32, _u64, _i32,
                                         _p, _p, _p, _p, _p, _p, _i64, _i32, _p]
        L.orc_classify_single.restype = _i32
        L.orc_classify_single.argtypes = [_p, _i32, _i32, _i32, _u64, _u64, _i32, _p, _i64, _p]
        L.orc_assemble_single.restype = _i32
        L.orc_assemble_single.argtypes = [_p, _i32, _i32, _u64, _u64, _i32, _i32, _p, _p]
        L.orc_ga_run.restype = _i64
        L.orc_ga_run.argtypes = [_p, _i64, _i32, _i32, _p, _u64, _i64, _i64, ctypes.c_uint32, _i64, _i32,
                                 _p, _p, _p, _i32]
        L.orc_ga_child.restype = _u64
        L.orc_ga_child.argtypes = [_u64, _i64, _i64, _p, _p, _i64, _i32, _i32, _p]
        L.orc_ga_draws.restype = None
        L.orc_ga_draws.argtypes = [_u64, _u64, _u64, _i64, _p]
        L.orc_ga_run_w.restype = _i64
        L.orc_ga_run_w.argtypes = [_p, _i64, _i32, _i32, _p, _u64, _i64, _i64, ctypes.c_uint32, _i64, _i32,
                                   _p, _p, _p, _i32]
        L.orc_ga_child_w.restype = None
        L.orc_ga_child_w.argtypes = [_u64, _i64, _i64, _p, _p, _i64, _i32, _i32, _p, _p]
        L.orc_ga_mutate.restype = _u64
        L.orc_ga_mutate.argtypes = [_p, _i64, _i32, _p, _u64, _i32, _u64, _i64, _i32]
        L.orc_ga_flip_counts.restype = None
        L.orc_ga_flip_counts.argtypes = [_u64, _i64, _i32, _p, _p]
        L.orc_stream_draws.restype = None
        L.orc_stream_draws.argtypes = [_u64, _u64, _u64, _i64, _p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def oat_hash_bytes(data) -> int:
    b = np.ascontiguousarray(np.asarray(data, dtype=np.uint8))
    return int(lib().orc_oat_hash_bytes(_ptr(b), b.shape[0]))


def stream_draws(seed: int, idx: int, run: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().orc_stream_draws(seed, idx, run, n, _ptr(out))
    return out


def classify_batch(indices, a, bpl, mask_pos, mask_val, free_pos, d, ks, hist_k, seed, strict,
                   out_class, out_hash, out_w, out_h, out_cells, out_shape,
                   nthreads: int = 0, counts: np.ndarray | None = None) -> None:
    """Same contract as tilevolve._kernels.classify_batch (_k:404-452)."""
    indices = np.ascontiguousarray(indices, dtype=np.uint64)
    mask_pos = np.ascontiguousarray(mask_pos, dtype=np.int64)
    mask_val = np.ascontiguousarray(mask_val, dtype=np.uint8)
    free_pos = np.ascontiguousarray(free_pos, dtype=np.int64)
    ks = np.ascontiguousarray(ks, dtype=np.int64)
    for arr, dt in ((out_class, np.uint8), (out_hash, np.uint32), (out_w, np.uint8),
                    (out_h, np.uint8), (out_cells, np.uint16), (out_shape, np.uint64)):
        assert arr.dtype == dt and arr.flags.c_contiguous
    cptr = None
    if counts is not None:
        assert counts.dtype == np.uint64 and counts.shape == (7,)
        cptr = _ptr(counts)
    rc = lib().orc_classify_batch(
        _ptr(indices), indices.shape[0], a, bpl, _ptr(mask_pos), _ptr(mask_val), mask_pos.shape[0],
        _ptr(free_pos), free_pos.shape[0], d, _ptr(ks), ks.shape[0], hist_k, int(seed), int(bool(strict)),
        _ptr(out_class), _ptr(out_hash), _ptr(out_w), _ptr(out_h), _ptr(out_cells), _ptr(out_shape),
        out_shape.shape[1], nthreads, cptr)
    if rc != 0:
        raise MemoryError("oracle scratch allocation failed")


def classify_single(edges, a, d, k, seed, genome_index, strict, shape_words):
    """(status, cls, hash, w, h, cells) as tilevolve._kernels.classify_single (_k:471-484)."""
    edges = np.ascontiguousarray(edges, dtype=np.uint8)
    out = np.zeros(5, np.int32)
    st = lib().orc_classify_single(_ptr(edges), a, d, k, int(seed), int(genome_index), int(bool(strict)),
                                   _ptr(shape_words), shape_words.shape[0], _ptr(out))
    return int(st), int(out[0]), int(np.uint32(np.int32(out[1]).view(np.uint32))), int(out[2]), int(out[3]), int(out[4])


def assemble_single(edges, a, d, seed, genome_index, run_index, strict, out_grid):
    """(outcome, minr, minc, maxr, maxc, n_placed) as tilevolve._kernels.assemble_single (_k:455-468)."""
    edges = np.ascontiguousarray(edges, dtype=np.uint8)
    out = np.zeros(6, np.int32)
    lib().orc_assemble_single(_ptr(edges), a, d, int(seed), int(genome_index), run_index, int(bool(strict)),
                              _ptr(out_grid), _ptr(out))
    return tuple(int(v) for v in out)


# ---------------------------------------------------------------- GA restatement (tv_ga_oracle.c)
def ga_run(pop: np.ndarray, L: int, mode: int, T: np.ndarray, seed: int, g0: int, n_gens: int, target: int,
           adapt_count: int, stop_when: int, nthreads: int = 0):
    """Runs in place on pop (u64); returns (gens_done, best u32, sum u64, count u32)."""
    assert pop.dtype == np.uint64 and pop.flags.c_contiguous
    T = np.ascontiguousarray(T, np.uint64)
    best = np.zeros(n_gens, np.uint32)
    sm = np.zeros(n_gens, np.uint64)
    cnt = np.zeros(n_gens, np.uint32)
    done = lib().orc_ga_run(_ptr(pop), pop.shape[0], L, mode, _ptr(T), int(seed), g0, n_gens, target, adapt_count,
                            stop_when, _ptr(best), _ptr(sm), _ptr(cnt), nthreads)
    return int(done), best[:done], sm[:done], cnt[:done]


def ga_child(seed, g, i, pop, cdf, L, mode, T) -> int:
    pop = np.ascontiguousarray(pop, np.uint64)
    cdf = np.ascontiguousarray(cdf, np.uint64)
    T = np.ascontiguousarray(T, np.uint64)
    return int(lib().orc_ga_child(int(seed), g, i, _ptr(pop), _ptr(cdf), pop.shape[0], L, mode, _ptr(T)))


def ga_draws(seed, g, i, n) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().orc_ga_draws(int(seed), g, i, n, _ptr(out))
    return out


def ga_flip_counts(seed, n, L, T) -> np.ndarray:
    out = np.empty(n, np.int32)
    T = np.ascontiguousarray(T, np.uint64)
    lib().orc_ga_flip_counts(int(seed), n, L, _ptr(T), _ptr(out))
    return out


def ga_run_w(pop: np.ndarray, L: int, mode: int, T: np.ndarray, seed: int, g0: int, n_gens: int, target: int,
             adapt_count: int, stop_when: int, nthreads: int = 0):
    """Wide genomes: pop u64 [n, W] (little-endian words), in place; as ga_run otherwise."""
    assert pop.dtype == np.uint64 and pop.flags.c_contiguous and pop.ndim == 2
    T = np.ascontiguousarray(T, np.uint64)
    best = np.zeros(n_gens, np.uint32)
    sm = np.zeros(n_gens, np.uint64)
    cnt = np.zeros(n_gens, np.uint32)
    done = lib().orc_ga_run_w(_ptr(pop), pop.shape[0], L, mode, _ptr(T), int(seed), g0, n_gens, target,
                              adapt_count, stop_when, _ptr(best), _ptr(sm), _ptr(cnt), nthreads)
    return int(done), best[:done], sm[:done], cnt[:done]


def ga_child_w(seed, g, i, pop, cdf, L, mode, T) -> np.ndarray:
    pop = np.ascontiguousarray(pop, np.uint64)
    cdf = np.ascontiguousarray(cdf, np.uint64)
    T = np.ascontiguousarray(T, np.uint64)
    out = np.zeros(pop.shape[1], np.uint64)
    lib().orc_ga_child_w(int(seed), g, i, _ptr(pop), _ptr(cdf), pop.shape[0], L, mode, _ptr(T), _ptr(out))
    return out


def ga_mutate(pop: np.ndarray, L: int, T: np.ndarray, pthr: int, method: int, seed: int, g: int,
              nthreads: int = 0) -> int:
    """SPEC ACCEPTANCE 8 operator benchmark (in place): method 0 by distribution, 1 bit by bit."""
    assert pop.dtype == np.uint64 and pop.flags.c_contiguous and pop.ndim == 2
    T = np.ascontiguousarray(T, np.uint64)
    return int(lib().orc_ga_mutate(_ptr(pop), pop.shape[0], L, _ptr(T), int(pthr), method, int(seed), g,
                                   nthreads))
