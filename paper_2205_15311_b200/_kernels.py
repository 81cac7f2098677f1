"""Drop-in for ``tilevolve._kernels`` (/root/reference/pkg/src/tilevolve/_kernels.py,
cited "_k:LINE"): same names, argument meaning, dtypes and in-place output
contract, executed by the sm_100a kernels in libtilevolve_b200.so.

Arrays may be numpy (host) or torch CUDA tensors (device, stream-ordered on
torch's current stream).  There is no CPU path: without the built library or
a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

# single-run outcomes (_k:19-22)
RUN_BOUNDED = 0
RUN_TRIVIAL = 1
RUN_UNBOUND = 2
RUN_OVERFLOW = 3
# classification codes (_k:25-29)
CLS_DETERMINISTIC = 0
CLS_TRIVIAL = 1
CLS_STERIC = 2
CLS_UNBOUND = 3
CLS_ERROR = 255

_OUT_DTYPES = (("out_class", np.uint8), ("out_hash", np.uint32), ("out_w", np.uint8), ("out_h", np.uint8),
               ("out_cells", np.uint16), ("out_shape", np.uint64))


def _host_arr(x, dtype):
    return np.ascontiguousarray(np.asarray(x), dtype=dtype)


def _check_out(name, arr, dtype, shape0):
    if isinstance(arr, np.ndarray):
        if arr.dtype != dtype or not arr.flags.c_contiguous:
            raise TypeError(f"{name} must be a C-contiguous {np.dtype(dtype).name} array")
        n0 = arr.shape[0]
    else:
        import torch
        tmap = {np.uint8: torch.uint8, np.uint16: torch.uint16, np.uint32: torch.uint32, np.uint64: torch.uint64}
        if arr.dtype != tmap[dtype] or not arr.is_contiguous() or not arr.is_cuda:
            raise TypeError(f"{name} must be a contiguous CUDA {np.dtype(dtype).name} tensor")
        n0 = arr.shape[0]
    if n0 != shape0:
        raise ValueError(f"{name} has {n0} rows, expected {shape0}")


def classify_batch(indices, a, bpl, mask_pos, mask_val, free_pos, d, ks, hist_k, seed, strict,
                   out_class, out_hash, out_w, out_h, out_cells, out_shape) -> None:
    """Classify a batch of enumeration indices (_k:404-452).

    ``ks`` is ascending; out_class[i, q] is the class the first ks[q] runs
    produce (prefix classification).  Hash / size / shape columns are the
    attribution at ``hist_k``; rows classified TRIVIAL/UNBOUND at hist_k get
    zero hash/w/h/cells and keep their out_shape row; capacity overflow sets
    every out_class column to 255 and writes nothing else.
    """
    L = _lib.lib()
    if _lib.is_cuda(indices):
        idx = indices.contiguous()
        n = idx.shape[0]
    else:
        idx = _host_arr(indices, np.uint64)
        n = idx.shape[0]
    ksa = _host_arr(ks, np.int64).reshape(-1)
    mp = _host_arr(mask_pos, np.int64).reshape(-1)
    mv = _host_arr(mask_val, np.uint8).reshape(-1)
    fp = _host_arr(free_pos, np.int64).reshape(-1)
    outs = (out_class, out_hash, out_w, out_h, out_cells, out_shape)
    for (name, dt), arr in zip(_OUT_DTYPES, outs):
        _check_out(name, arr, dt, n)
    q = ksa.shape[0]
    if tuple(out_class.shape[1:]) != (q,):
        raise ValueError(f"out_class must be (n, {q})")
    if len(out_shape.shape) != 2:
        raise ValueError("out_shape must be (n, W)")
    W = int(out_shape.shape[1])
    with _lib.device_of(idx, *outs):  # device tensors: run on their device, on its current stream
        stream = _lib.stream_of(idx, *outs)
        _lib.check(L.tv_classify_batch(
            _lib.ptr(idx), n, int(a), int(bpl), _lib.ptr(mp), _lib.ptr(mv), mp.shape[0], _lib.ptr(fp), fp.shape[0],
            int(d), _lib.ptr(ksa), q, int(hist_k), int(np.uint64(seed)), int(bool(strict)),
            *[_lib.ptr(o) for o in outs], W, stream))


def assemble_single(edges, a, d, seed, genome_index, run_index, strict, out_grid):
    """One assembly run with the grid copied out (_k:455-468).
    Returns (outcome, minr, minc, maxr, maxc, n_placed)."""
    e = _host_arr(edges, np.uint8)
    if not (isinstance(out_grid, np.ndarray) and out_grid.dtype == np.int16 and out_grid.flags.c_contiguous
            and out_grid.size == d * d):
        raise TypeError("out_grid must be a C-contiguous int16 array of d*d cells")
    out = (ctypes.c_int32 * 6)()
    _lib.check(_lib.lib().tv_assemble_single(_lib.ptr(e), int(a), int(d), int(np.uint64(seed)),
                                             int(np.uint64(genome_index)), int(run_index), int(bool(strict)),
                                             _lib.ptr(out_grid), out))
    return tuple(int(v) for v in out)


def classify_single(edges, a, d, k, seed, genome_index, strict, shape_words):
    """Classify one tile set (_k:471-484).  Returns (status, cls, hash, w, h, cells);
    shape_words is written as the reference writes it."""
    e = _host_arr(edges, np.uint8)
    if not (isinstance(shape_words, np.ndarray) and shape_words.dtype == np.uint64
            and shape_words.flags.c_contiguous):
        raise TypeError("shape_words must be a C-contiguous uint64 array")
    out = (ctypes.c_int32 * 6)()
    _lib.check(_lib.lib().tv_classify_single(_lib.ptr(e), int(a), int(d), int(k), int(np.uint64(seed)),
                                             int(np.uint64(genome_index)), int(bool(strict)), _lib.ptr(shape_words),
                                             shape_words.shape[0], out))
    return (int(out[0]), int(out[1]), np.uint32(out[2] & 0xFFFFFFFF), int(out[3]), int(out[4]), int(out[5]))


def oat_hash_bytes(data) -> np.uint32:
    """32-bit one-at-a-time hash of a uint8 array (_k:79-85)."""
    b = _host_arr(data, np.uint8).reshape(-1)
    out = ctypes.c_uint32()
    _lib.check(_lib.lib().tv_oat_hash_bytes(_lib.ptr(b), b.shape[0], ctypes.byref(out)))
    return np.uint32(out.value)


def edges_from_labels(labels: np.ndarray, a: int) -> np.ndarray:
    """In-situ edge table edges[t*16 + orient*4 + dir] from flat N,E,S,W labels (_k:487-494)."""
    lab = np.asarray(labels).reshape(a, 4)
    rt = np.arange(4)[:, None]
    dr = np.arange(4)[None, :]
    src = (dr - rt) & 3                      # [orient, dir] -> original edge
    return lab[:, src].reshape(a * 16).astype(np.uint8)
