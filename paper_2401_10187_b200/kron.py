"""ctypes binding of libkron (include/kron.h).  Argument marshalling only — every step of the
Kron-Matmul path runs in the library's CUDA kernels.  Names follow the C-ABI."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(HERE, "libkron.so")

if not os.path.exists(lib_path):
    raise ImportError(f"libkron.so not built ({lib_path}); run `python -m paper_2401_10187_b200.build` "
                      "(or __graft_entry__.build()). There is no CPU fallback.")

_lib = ctypes.CDLL(lib_path)

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vpp = ctypes.POINTER(ctypes.c_void_p)

STATUS = {0: "KRON_OK", 1: "KRON_ERR_INVALID_ARG", 2: "KRON_ERR_SHAPE", 3: "KRON_ERR_UNSUPPORTED",
          4: "KRON_ERR_NO_MEMORY", 5: "KRON_ERR_CUDA", 6: "KRON_ERR_NCCL", 7: "KRON_ERR_DIST_LAYOUT"}

_lib.kron_status_string.restype = ctypes.c_char_p
_lib.kron_status_string.argtypes = [ctypes.c_int]
_lib.kron_matmul.restype = ctypes.c_int
_lib.kron_matmul.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_void_p, _vpp, ctypes.c_void_p,
                             ctypes.c_int, ctypes.c_void_p]
_lib.kron_matmul_ws.restype = ctypes.c_int
_lib.kron_matmul_ws.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_void_p, _vpp, ctypes.c_void_p,
                                ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
_lib.kron_matmul_ws_events.restype = ctypes.c_int
_lib.kron_matmul_ws_events.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_void_p, _vpp,
                                       ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, _vpp,
                                       ctypes.c_int32, ctypes.c_void_p]
_lib.kron_matmul_workspace_size.restype = ctypes.c_int
_lib.kron_matmul_workspace_size.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_size_t)]
_lib.kron_plan_describe.restype = ctypes.c_int
_lib.kron_plan_describe.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int, ctypes.c_int32,
                                    _i32p, _i32p, _i32p, _i32p]
_lib.kron_plan_cost.restype = ctypes.c_int
_lib.kron_plan_cost.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int,
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
_lib.kron_dist_plan.restype = ctypes.c_int
_lib.kron_dist_plan.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int32, _i32p, _i32p, _i64p]
_lib.kron_dist_grid_rule.restype = ctypes.c_int
_lib.kron_dist_grid_rule.argtypes = [ctypes.c_int32, _i32p, _i32p]

KIND_NAMES = {0: "generic", 1: "fused", 2: "gemm"}


class KronError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {STATUS.get(code, code)}")


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise KronError(rc, what)


def dtype_code(dtype) -> int:
    s = str(dtype)
    if s.endswith("float32"):
        return 0
    if s.endswith("float64"):
        return 1
    raise TypeError(f"Kron-Matmul supports float32 and float64, got {dtype}")


def _shape_arrays(P, Q):
    n = len(P)
    return (ctypes.c_int32 * n)(*[int(p) for p in P]), (ctypes.c_int32 * n)(*[int(q) for q in Q])


def _stream_ptr(stream) -> int:
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def workspace_size(M: int, P, Q, dtype) -> int:
    Pa, Qa = _shape_arrays(P, Q)
    out = ctypes.c_size_t()
    _check(_lib.kron_matmul_workspace_size(M, len(P), Pa, Qa, dtype_code(dtype), ctypes.byref(out)),
           "kron_matmul_workspace_size")
    return int(out.value)


def plan_describe(M: int, P, Q, dtype):
    """[(first factor (1-based), number fused, kernel family)] of the pass plan kron_matmul uses."""
    Pa, Qa = _shape_arrays(P, Q)
    cap = 64
    n = ctypes.c_int32()
    first = (ctypes.c_int32 * cap)()
    nf = (ctypes.c_int32 * cap)()
    kind = (ctypes.c_int32 * cap)()
    _check(_lib.kron_plan_describe(M, len(P), Pa, Qa, dtype_code(dtype), cap, ctypes.byref(n), first, nf, kind),
           "kron_plan_describe")
    return [(first[i], nf[i], KIND_NAMES[kind[i]]) for i in range(n.value)]


def plan_cost(M: int, P, Q, dtype):
    """(algorithmic HBM bytes, FLOPs) of the plan."""
    Pa, Qa = _shape_arrays(P, Q)
    b, f = ctypes.c_double(), ctypes.c_double()
    _check(_lib.kron_plan_cost(M, len(P), Pa, Qa, dtype_code(dtype), ctypes.byref(b), ctypes.byref(f)),
           "kron_plan_cost")
    return b.value, f.value


def dist_plan(M: int, P, Q, GM: int, GK: int):
    """(rounds, ledger) of the distributed round plan (host only)."""
    Pa, Qa = _shape_arrays(P, Q)
    cap = 64
    n = ctypes.c_int32()
    rounds = (ctypes.c_int32 * cap)()
    ledger = (ctypes.c_int64 * cap)()
    _check(_lib.kron_dist_plan(M, len(P), Pa, Qa, GM, GK, cap, ctypes.byref(n), rounds, ledger), "kron_dist_plan")
    return [rounds[i] for i in range(n.value)], [ledger[i] for i in range(n.value)]


def grid_rule(G: int):
    gm, gk = ctypes.c_int32(), ctypes.c_int32()
    _check(_lib.kron_dist_grid_rule(G, ctypes.byref(gm), ctypes.byref(gk)), "kron_dist_grid_rule")
    return gm.value, gk.value


def _prep(X, Fs):
    if X.dim() != 2:
        raise ValueError("X must be 2-D (M x prod P)")
    if not X.is_cuda or not X.is_contiguous():
        raise ValueError("X must be a contiguous CUDA tensor")
    P = [int(f.shape[0]) for f in Fs]
    Q = [int(f.shape[1]) for f in Fs]
    for f in Fs:
        if not f.is_cuda or not f.is_contiguous() or f.dtype != X.dtype or f.dim() != 2:
            raise ValueError("factors must be contiguous 2-D CUDA tensors of X's dtype")
    K = 1
    for p in P:
        K *= p
    if X.shape[1] != K:
        raise ValueError(f"X has {X.shape[1]} columns, prod P = {K}")
    return P, Q


def matmul(X, Fs, out=None, stream=None):
    """Y = X · (F^1 ⊗ … ⊗ F^N) on the current (or given) CUDA stream via kron_matmul()."""
    import torch
    P, Q = _prep(X, Fs)
    L = 1
    for q in Q:
        L *= q
    if out is None:
        out = torch.empty((X.shape[0], L), dtype=X.dtype, device=X.device)
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    _check(_lib.kron_matmul(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(), dtype_code(X.dtype),
                            _stream_ptr(stream)), "kron_matmul")
    return out


def matmul_ws(X, Fs, out, workspace, stream=None):
    """kron_matmul_ws(): caller-owned output and workspace (a uint8 CUDA tensor, or None if 0 bytes)."""
    P, Q = _prep(X, Fs)
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    wptr = workspace.data_ptr() if workspace is not None else None
    wbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(_lib.kron_matmul_ws(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(), dtype_code(X.dtype),
                               wptr, wbytes, _stream_ptr(stream)), "kron_matmul_ws")
    return out


def matmul_ws_events(X, Fs, out, workspace, events, stream=None):
    """kron_matmul_ws_events(): like matmul_ws, recording events[i] (raw cudaEvent_t handles) before
    pass i and events[npasses] after the last pass, for per-kernel timing."""
    P, Q = _prep(X, Fs)
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    Ev = (ctypes.c_void_p * len(events))(*[int(e) for e in events])
    wptr = workspace.data_ptr() if workspace is not None else None
    wbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(_lib.kron_matmul_ws_events(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(),
                                      dtype_code(X.dtype), wptr, wbytes, Ev, len(events), _stream_ptr(stream)),
           "kron_matmul_ws_events")
    return out


def raw_lib():
    return _lib
