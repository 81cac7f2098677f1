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
