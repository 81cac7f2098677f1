"""Loader for libtilevolve_b200.so (the C ABI in include/tilevolve_b200.h).

The product path is CUDA only: if the shared library is missing or no CUDA
device is usable, calls raise -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libtilevolve_b200.so")
CSRC = os.path.join(PKG_DIR, "csrc")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

_lib = None


class TvError(RuntimeError):
    """Error reported by libtilevolve_b200 (tv_last_error)."""


def build(verbose: bool = False) -> str:
    """Compile every CUDA source into the in-tree shared library for sm_100a."""
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(os.path.join(CSRC, "tv_capi.cu")):
        raise FileNotFoundError(CSRC)
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB_PATH, os.path.join(CSRC, "tv_capi.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return LIB_PATH


_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64

_SIGS = {
    "tv_version": (_i32, []),
    "tv_last_error": (ctypes.c_char_p, []),
    "tv_last_launch_info": (_i32, [_p]),
    "tv_classify_batch": (_i32, [_p, _i64, _i32, _i32, _p, _p, _i64, _p, _i64, _i32, _p, _i64, _i32, _u64, _i32,
                                 _p, _p, _p, _p, _p, _p, _i64, _p]),
    "tv_classify_single": (_i32, [_p, _i32, _i32, _i32, _u64, _u64, _i32, _p, _i64, _p]),
    "tv_assemble_single": (_i32, [_p, _i32, _i32, _u64, _u64, _i32, _i32, _p, _p]),
    "tv_oat_hash_bytes": (_i32, [_p, _i64, _p]),
    "tv_shape_labels": (_i32, [_p, _p, _p, _i64, _i64, _p, _p, _p]),
    "tv_hist_create": (_i32, [_i64, _i32, _i32, ctypes.POINTER(_p)]),
    "tv_hist_destroy": (_i32, [_p]),
    "tv_hist_clear": (_i32, [_p, _p]),
    "tv_hist_count": (_i32, [_p, _p, _p, _p]),
    "tv_hist_export": (_i32, [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "tv_hist_pack": (_i32, [_p, _i64, _p, _p, _p, _p]),
    "tv_hist_replace_rows": (_i32, [_p, _i64, _p, _p, _p]),
    "tv_hist_merge": (_i32, [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "tv_enumerate_range": (_i32, [_u64, _u64, _i32, _i32, _p, _p, _i64, _p, _i64, _i32, _p, _i64, _i32, _u64, _i32,
                                  _p, _p]),
    "tv_enumerate_chunks": (_i32, [_u64, _u64, _u64, _u64, _i32, _i32, _p, _p, _i64, _p, _i64, _i32, _p, _i64, _i32,
                                   _u64, _i32, _p, _p]),
    "tv_enumerate_indices": (_i32, [_p, _i64, _i32, _i32, _p, _p, _i64, _p, _i64, _i32, _p, _i64, _i32, _u64, _i32,
                                    _p, _p]),
    "tv_ga_create": (_i32, [_i64, _i32, _i32, _p, ctypes.POINTER(_p)]),
    "tv_ga_destroy": (_i32, [_p]),
    "tv_ga_set_population": (_i32, [_p, _p, _p]),
    "tv_ga_get_population": (_i32, [_p, _p, _p]),
    "tv_ga_population_ptr": (_i32, [_p, ctypes.POINTER(_p)]),
    "tv_ga_run": (_i32, [_p, _u64, _i64, _i64, ctypes.c_uint32, _i64, _i32, _p, _p, _p, _p, _p, _p]),
    "tv_ga_replicas": (_i32, [_i64, _i32, _i32, _p, _i32, _p, _p, _i64, _i64, ctypes.c_uint32, _i64, _i32, _p, _p, _p,
                              _p, _p, _p, _p, _p]),
    "tv_ga_fitness_jatam": (_i32, [_p, _i32, _i32, _p, _p, _i64, _p, _i64, _i32, _i32, _u64, _i32, _p, _p, _p]),
    "tv_ga_mutate": (_i32, [_p, _i64, _i32, _p, _u64, _i32, _u64, _i64, _p, _p]),
    "tv_ga_run_jatam": (_i32, [_p, _i32, _i32, _p, _p, _i64, _p, _i64, _i32, _i32, _u64, _i32, _p, _u64, _i64, _i64,
                               ctypes.c_uint32, _p, _p, _p, _p]),
    "tv_int_peak_launch": (_i32, [_i64, _i32, _i32, _p, _p]),
    "tv_sm_count": (_i32, [_p]),
    "tv_l2_probe_launch": (_i32, [_p, _i64, _i32, _i32, _p, _p]),
    "tv_gridsync_probe_launch": (_i32, [_i32, _p]),
}


def exported_symbols() -> list[str]:
    return list(_SIGS)


def lib():
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        path = os.environ.get("TV_LIB_PATH", LIB_PATH)  # alternate build for A/B measurements
        if not os.path.exists(path):
            raise TvError(f"CUDA extension missing: {path} (run __graft_entry__.build())")
        L = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().tv_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise TvError(f"libtilevolve_b200 error {rc}: {msg}")


def ptr(a):
    """Raw address of a numpy array (host) or a torch tensor (host or CUDA)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    raise TypeError(f"expected numpy array or torch tensor, got {type(a).__name__}")


def is_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def stream_of(*arrays):
    """cudaStream_t for a call: torch's current stream when any argument is a CUDA tensor."""
    for a in arrays:
        if is_cuda(a):
            import torch
            return ctypes.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)
    return None


def device_of(*arrays):
    """Context that makes the CUDA tensors' device current for a call (a no-op for host
    arrays); tensors on different devices are refused."""
    import contextlib
    devs = {a.device.index for a in arrays if is_cuda(a)}
    if not devs:
        return contextlib.nullcontext()
    if len(devs) > 1:
        raise ValueError(f"CUDA tensors on different devices {sorted(devs)}")
    import torch
    return torch.cuda.device(devs.pop())


def launch_info() -> dict:
    info = (ctypes.c_int64 * 5)()
    lib().tv_last_launch_info(info)
    return dict(path={1: "bitboard", 2: "generic", 3: "ga"}.get(info[0], "none"), ctas=info[1], threads=info[2],
                smem=info[3], launches=info[4])
