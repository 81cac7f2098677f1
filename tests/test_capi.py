"""The C-ABI library loads without a GPU and exports every symbol the header declares."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib_path():
    from paper_2205_15311_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.LIB_PATH


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tilevolve_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*\**(tv_[a-z_0-9]+)\s*\(", src, re.M)))


def test_header_declares_core_entry_points():
    syms = header_symbols()
    for s in ("tv_classify_batch", "tv_classify_single", "tv_assemble_single", "tv_oat_hash_bytes",
              "tv_enumerate_range", "tv_hist_export", "tv_hist_merge"):
        assert s in syms


def test_library_exports_every_header_symbol():
    L = ctypes.CDLL(_lib_path())
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_python_signatures_cover_header():
    from paper_2205_15311_b200 import _lib
    assert set(header_symbols()) <= set(_lib.exported_symbols())


def test_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2205_15311_b200 import _kernels, _lib
    _lib_path()
    with pytest.raises(_lib.TvError):
        _kernels.oat_hash_bytes(np.array([1, 2, 3], np.uint8))


def test_argument_validation_is_host_side():
    """Bad arguments are rejected before any device work (ValueError, like numba's typing errors)."""
    from paper_2205_15311_b200 import _kernels, _lib
    _lib_path()
    n = 4
    outs = [np.zeros((n, 1), np.uint8), np.zeros(n, np.uint32), np.zeros(n, np.uint8), np.zeros(n, np.uint8),
            np.zeros(n, np.uint16), np.zeros((n, 6), np.uint64)]
    with pytest.raises(TypeError):
        _kernels.classify_batch(np.arange(n, dtype=np.uint64), 2, 3, [], [], np.arange(23, -1, -1), 19, [8], 8, 0,
                                True, outs[0].astype(np.int8), *outs[1:])


def test_enumeration_rejects_indices_past_the_space():
    """Index bits >= nfree are ignored by the decoder, so a range past 2^nfree would alias
    genomes (idx mod 2^nfree) and count them twice: rejected before any device work."""
    from paper_2205_15311_b200 import _lib
    from paper_2205_15311_b200.classify import enumerate_space
    from paper_2205_15311_b200.genome import SearchSpace
    _lib_path()
    L = _lib.lib()
    a, bpl, mp, mv, fp = SearchSpace(2, 8).kernel_args()
    ks = np.array([8], np.int64)
    P = _lib.ptr
    for start, count in (((1 << 24) - 10, 11), (1 << 24, 1), (2 ** 64 - 2, 5)):
        rc = L.tv_enumerate_range(start, count, a, bpl, P(mp), P(mv), mp.shape[0], P(fp), fp.shape[0], 19, P(ks), 1,
                                  8, 0, 1, None, None)
        assert rc == -1 and (b"outside the space" in L.tv_last_error() or b"wraps" in L.tv_last_error())
    # chunks: 3 chunks of 2^20 at stride 2^23 from 2^20 end at 2^20 + 2 * 2^23 + 2^20 > 2^24
    rc = L.tv_enumerate_chunks(1 << 20, 3 << 20, 1 << 20, 1 << 23, a, bpl, P(mp), P(mv), mp.shape[0], P(fp),
                               fp.shape[0], 19, P(ks), 1, 8, 0, 1, None, None)
    assert rc == -1 and b"outside the space" in L.tv_last_error()
    # in range: fails later, on the null histogram, not on the range
    rc = L.tv_enumerate_chunks(0, 2 << 20, 1 << 20, 1 << 23, a, bpl, P(mp), P(mv), mp.shape[0], P(fp), fp.shape[0],
                               19, P(ks), 1, 8, 0, 1, None, None)
    assert rc == -1 and b"null histogram" in L.tv_last_error()
    with pytest.raises(ValueError):
        enumerate_space(SearchSpace(2, 8), ks=(8,), start=(1 << 24) - 10, count=20)
