"""oracle — the CPU oracle for Kron-Matmul (arxiv 2401.10187).  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this package.  It shares no code with the CUDA path
(``paper_2401_10187_b200``) and neither imports the other.  The arithmetic lives in plain C
(``kron_oracle.c``, fp64, ``-O2 -ffp-contract=off``); this module only marshals numpy arrays.

Functions (each cites the passage it follows in kron_oracle.c):
    kron_product   O1  Kronecker definition
    naive          O1  materialise + dense matmul            [K*L <= 2^26]
    sliced_multiply    one iteration of Algorithm 1
    widths             intermediate widths (Alg 1, reading G2)
    alg1           O2  Algorithm 1 on all rows or a row subset
    alg2           O3  Algorithm 2 simulated on {GM,GK} GPUs + ledger
    fused_store_col    Fig 7 StoreFusedShMem index map (reading G7)
    shift_pos          Fig 5 shift-caching position (reading G6)
    grid               GPU grid rule

Parity status: every function above is pinned by tests/test_oracle.py against values the paper
prints, closed forms, identities and brute force; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "kron_oracle.c")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_L = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> None:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
                               "-shared", "-o", LIB, SRC])


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB)
        _lib.oracle_kron_product.argtypes = [ctypes.c_int, _I, _I, ctypes.POINTER(_D), _D]
        _lib.oracle_naive.argtypes = [ctypes.c_int64, ctypes.c_int, _I, _I, _D, ctypes.POINTER(_D), _D]
        _lib.oracle_sliced_multiply.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _D, _D, _D]
        _lib.oracle_widths.argtypes = [ctypes.c_int, _I, _I, _L]
        _lib.oracle_alg1.argtypes = [ctypes.c_int64, ctypes.c_int, _I, _I, _D, ctypes.POINTER(_D), _D]
        _lib.oracle_fused_store_col.restype = ctypes.c_int64
        _lib.oracle_fused_store_col.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                                ctypes.c_int64, ctypes.c_int64]
        _lib.oracle_threads.restype = ctypes.c_int
        _lib.oracle_threads.argtypes = [ctypes.c_int]
        _lib.oracle_shift_pos.restype = ctypes.c_int64
        _lib.oracle_shift_pos.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        _lib.oracle_grid.argtypes = [ctypes.c_int, _I, _I]
        _lib.oracle_alg2.argtypes = [ctypes.c_int64, ctypes.c_int, _I, _I, _D, ctypes.POINTER(_D), ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, _I, _D, _L]
    return _lib


def _ints(v):
    a = (ctypes.c_int * len(v))(*[int(x) for x in v])
    return a


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _factor_ptrs(Fs):
    Fs = [_f64(f) for f in Fs]
    arr = (_D * len(Fs))(*[f.ctypes.data_as(_D) for f in Fs])
    return Fs, arr


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def shapes(Fs):
    return [int(f.shape[0]) for f in Fs], [int(f.shape[1]) for f in Fs]


def kron_product(Fs) -> np.ndarray:
    P, Q = shapes(Fs)
    keep, arr = _factor_ptrs(Fs)
    G = np.empty((int(np.prod(P)), int(np.prod(Q))), dtype=np.float64)
    _check(lib().oracle_kron_product(len(P), _ints(P), _ints(Q), arr, G.ctypes.data_as(_D)), "kron_product")
    return G


def naive(X, Fs) -> np.ndarray:
    X = _f64(X)
    P, Q = shapes(Fs)
    keep, arr = _factor_ptrs(Fs)
    Y = np.empty((X.shape[0], int(np.prod(Q))), dtype=np.float64)
    _check(lib().oracle_naive(X.shape[0], len(P), _ints(P), _ints(Q), X.ctypes.data_as(_D), arr,
                              Y.ctypes.data_as(_D)), "naive")
    return Y


def sliced_multiply(T, F) -> np.ndarray:
    T = _f64(T)
    F = _f64(F)
    rows, K = T.shape
    P, Q = F.shape
    Y = np.empty((rows, K // P * Q), dtype=np.float64)
    _check(lib().oracle_sliced_multiply(rows, K, P, Q, T.ctypes.data_as(_D), F.ctypes.data_as(_D),
                                        Y.ctypes.data_as(_D)), "sliced_multiply")
    return Y


def widths(P, Q):
    W = (ctypes.c_int64 * (len(P) + 1))()
    _check(lib().oracle_widths(len(P), _ints(P), _ints(Q), W), "widths")
    return [int(w) for w in W]


def alg1(X, Fs) -> np.ndarray:
    """O2 Algorithm 1 on the rows of X (X may be a row subset of the full input)."""
    X = _f64(X)
    P, Q = shapes(Fs)
    keep, arr = _factor_ptrs(Fs)
    Y = np.empty((X.shape[0], int(np.prod(Q))), dtype=np.float64)
    _check(lib().oracle_alg1(X.shape[0], len(P), _ints(P), _ints(Q), X.ctypes.data_as(_D), arr,
                             Y.ctypes.data_as(_D)), "alg1")
    return Y


def alg2(X, Fs, GM: int, GK: int, local):
    """O3 Algorithm 2 simulation.  Returns (Y gathered, per-round ledger list)."""
    X = _f64(X)
    P, Q = shapes(Fs)
    keep, arr = _factor_ptrs(Fs)
    Y = np.empty((X.shape[0], int(np.prod(Q))), dtype=np.float64)
    ledger = (ctypes.c_int64 * len(local))()
    _check(lib().oracle_alg2(X.shape[0], len(P), _ints(P), _ints(Q), X.ctypes.data_as(_D), arr, GM, GK,
                             len(local), _ints(local), Y.ctypes.data_as(_D), ledger), "alg2")
    return Y, [int(v) for v in ledger]


def fused_store_col(K, P, TileK, Fused, bidy, c) -> int:
    return int(lib().oracle_fused_store_col(K, P, TileK, Fused, bidy, c))


def shift_pos(k, TileP, RegK) -> int:
    return int(lib().oracle_shift_pos(k, TileP, RegK))


def grid(G: int):
    gm, gk = ctypes.c_int(), ctypes.c_int()
    rc = lib().oracle_grid(G, ctypes.byref(gm), ctypes.byref(gk))
    if rc != 0:
        return None
    return gm.value, gk.value


def threads(n: int = 0) -> int:
    """OpenMP threads of the row-parallel loops: n > 0 sets the count (torchrun exports
    OMP_NUM_THREADS=1 to every rank); returns the count in effect.  Results do not depend on it."""
    return int(lib().oracle_threads(int(n)))
