"""synth — seeded, counter-based synthetic inputs for the Kron-Matmul path.

Test and bench infrastructure shared by the oracle side and the CUDA side.  It holds none of
the method's arithmetic: it only produces X and the factors F^i (
SURVEY.md §8(d) d.3).  Two twins implement the same generator: ``synth.c`` (host, OpenMP) and
``synth_dev.cu`` (device fill kernel).  ``tests/test_synth.py`` pins them to each other and to
the published splitmix64 reference values.

Seeds: ``SEED_BASE + cfg`` (A=0, B=1, C=2, D1=3, D2=4, E=5).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_HOST = os.path.join(HERE, "libsynth.so")
LIB_DEV = os.path.join(HERE, "libsynth_dev.so")
SEED_BASE = 240110187
MODES = {"urand": 0, "srand": 1, "int": 2, "int1": 3}
NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

_host = None
_dev = None


def build(force: bool = False) -> None:
    """Compile the host twin with gcc and the device twin with nvcc (sm_100a)."""
    src = os.path.join(HERE, "synth.c")
    if force or not os.path.exists(LIB_HOST) or os.path.getmtime(LIB_HOST) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", LIB_HOST, src])
    dsrc = os.path.join(HERE, "synth_dev.cu")
    if force or not os.path.exists(LIB_DEV) or os.path.getmtime(LIB_DEV) < os.path.getmtime(dsrc):
        subprocess.check_call(["nvcc", *NVCC_ARCH, "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
                               "-o", LIB_DEV, dsrc])


def _lib_host():
    global _host
    if _host is None:
        if not os.path.exists(LIB_HOST):
            build()
        _host = ctypes.CDLL(LIB_HOST)
        _host.synth_splitmix64.restype = ctypes.c_uint64
        _host.synth_splitmix64.argtypes = [ctypes.c_uint64]
        for name, ct in (("synth_fill_f64", ctypes.c_double), ("synth_fill_f32", ctypes.c_float)):
            fn = getattr(_host, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.POINTER(ct), ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                           ctypes.c_uint64, ctypes.c_int]
        _host.synth_fill_rows_f64.restype = ctypes.c_int
        _host.synth_fill_rows_f64.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                                              ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                              ctypes.c_uint64, ctypes.c_int]
    return _host


def _lib_dev():
    global _dev
    if _dev is None:
        if not os.path.exists(LIB_DEV):
            build()
        _dev = ctypes.CDLL(LIB_DEV)
        for name in ("synth_fill_block_dev_f32", "synth_fill_block_dev_f64"):
            fn = getattr(_dev, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                           ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
    return _dev


def splitmix64(x: int) -> int:
    return int(_lib_host().synth_splitmix64(ctypes.c_uint64(x & (2**64 - 1))))


def fill(n: int, seed: int, tensor_id: int, mode: str = "urand", dtype=np.float64, first: int = 0) -> np.ndarray:
    """n consecutive elements (linear index first..first+n) of tensor `tensor_id`."""
    lib = _lib_host()
    dt = np.dtype(dtype)
    out = np.empty(n, dtype=dt)
    if dt == np.float64:
        rc = lib.synth_fill_f64(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, first, seed, tensor_id, MODES[mode])
    elif dt == np.float32:
        rc = lib.synth_fill_f32(out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n, first, seed, tensor_id, MODES[mode])
    else:
        raise TypeError(dt)
    if rc != 0:
        raise RuntimeError("synth fill failed")
    return out


def matrix(rows: int, cols: int, seed: int, tensor_id: int, mode: str = "urand", dtype=np.float64) -> np.ndarray:
    return fill(rows * cols, seed, tensor_id, mode, dtype).reshape(rows, cols)


def rows_of(rows, cols: int, seed: int, tensor_id: int = 0, mode: str = "urand") -> np.ndarray:
    """Selected rows (fp64) of the implicit rows x cols matrix: the oracle's row-subset input."""
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    out = np.empty((len(r), cols), dtype=np.float64)
    rc = _lib_host().synth_fill_rows_f64(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                         r.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(r), cols,
                                         seed, tensor_id, MODES[mode])
    if rc != 0:
        raise RuntimeError("synth rows failed")
    return out


def gp_factor(P: int, Q: int) -> np.ndarray:
    """RBF kernel-matrix factor on a 1-D grid (SKI-style K^i), fp64.

    square: F[i,j] = exp(-(i-j)^2 / (2 l^2)), l = P/8;  non-square: grid i/(P-1) vs j/(Q-1), l = 0.1.
    """
    i = np.arange(P, dtype=np.float64)[:, None]
    j = np.arange(Q, dtype=np.float64)[None, :]
    if P == Q:
        ell = max(P / 8.0, 0.5)
        return np.exp(-((i - j) ** 2) / (2 * ell * ell))
    a = i / max(P - 1, 1)
    b = j / max(Q - 1, 1)
    return np.exp(-((a - b) ** 2) / (2 * 0.1 * 0.1))


def factors(P, Q, seed: int, mode: str = "urand", dtype=np.float64):
    """Factors F^1..F^N (tensor ids 1..N), host arrays. mode 'gp' gives RBF factors."""
    out = []
    for i, (p, q) in enumerate(zip(P, Q)):
        if mode == "gp":
            out.append(gp_factor(p, q).astype(dtype))
        else:
            out.append(matrix(p, q, seed, i + 1, mode, dtype))
    return out


def fill_device(ptr: int, rows: int, cols: int, seed: int, tensor_id: int, mode: str, dtype,
                stream: int = 0, r0: int = 0, c0: int = 0, ld: int | None = None) -> None:
    """Generate X[r0:r0+rows, c0:c0+cols] (of a matrix with `ld` columns) straight into device memory."""
    lib = _lib_dev()
    dt = np.dtype(dtype)
    fn = lib.synth_fill_block_dev_f32 if dt == np.float32 else lib.synth_fill_block_dev_f64
    rc = fn(ptr, rows, cols, r0, c0, cols if ld is None else ld, seed, tensor_id, MODES[mode], stream)
    if rc != 0:
        raise RuntimeError(f"synth device fill failed rc={rc}")


def row_subset(M: int, extra: int = 60, seed: int = 0):
    """Rows {0, 1, M/2, M-1} plus `extra` seeded rows."""
    base = {0, min(1, M - 1), M // 2, M - 1}
    rng = np.random.default_rng(seed + 7)
    if M > len(base):
        more = rng.choice(M, size=min(extra, M), replace=False)
        base.update(int(x) for x in more)
    return np.array(sorted(r for r in base if 0 <= r < M), dtype=np.int64)


__all__ = ["build", "splitmix64", "fill", "matrix", "rows_of", "gp_factor", "factors", "fill_device",
           "row_subset", "SEED_BASE", "MODES"]
