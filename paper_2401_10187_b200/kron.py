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
_lib.kron_last_error_detail.restype = ctypes.c_char_p
_lib.kron_last_error_detail.argtypes = []
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

_lib.kron_autotune.restype = ctypes.c_int
_lib.kron_autotune.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_void_p, _vpp, ctypes.c_void_p,
                               ctypes.c_int, ctypes.c_int32, ctypes.c_void_p, _i32p, ctypes.POINTER(ctypes.c_float)]
_lib.kron_autotune_candidates.restype = ctypes.c_int
_lib.kron_autotune_candidates.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int, _i32p]
_lib.kron_plan_kernel.restype = ctypes.c_int
_lib.kron_plan_kernel.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int, ctypes.c_int32,
                                  ctypes.c_char_p, ctypes.c_int32]
_lib.kron_plan_cache_clear.restype = ctypes.c_int
_lib.kron_plan_cache_clear.argtypes = []

_lib.kron_graph_create.restype = ctypes.c_int
_lib.kron_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_void_p, _vpp, ctypes.c_void_p,
                                   ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
_lib.kron_graph_launch.restype = ctypes.c_int
_lib.kron_graph_launch.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
_lib.kron_graph_destroy.restype = ctypes.c_int
_lib.kron_graph_destroy.argtypes = [ctypes.c_void_p]

_lib.kron_matmul_host.restype = ctypes.c_int
_lib.kron_matmul_host.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_void_p, _vpp, ctypes.c_void_p,
                                  ctypes.c_int, ctypes.c_int64, ctypes.c_void_p]

KIND_NAMES = {0: "generic", 1: "fused", 2: "gemm", 3: "chain"}


class KronError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        detail = _lib.kron_last_error_detail().decode() if code in (5, 6) else ""
        super().__init__(f"{what}: {STATUS.get(code, code)}" + (f" ({detail})" if detail else ""))


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise KronError(rc, what)


MODES = {None: None, "fp32": None, "3xtf32": 2, "tf32": 3}


def dtype_code(dtype, mode=None) -> int:
    """C-ABI dtype: 0 float32, 1 float64; float32 data in the separately reported tensor-core modes:
    2 (mode="3xtf32", split operands, ~fp32 accuracy) and 3 (mode="tf32", plain TF32 products)."""
    s = str(dtype)
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r} (None, 'tf32' or '3xtf32')")
    if s.endswith("float32"):
        return MODES[mode] if MODES[mode] is not None else 0
    if mode is not None and MODES[mode] is not None:
        raise ValueError("the tensor-core modes apply to float32 data only")
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


def workspace_size(M: int, P, Q, dtype, mode=None) -> int:
    Pa, Qa = _shape_arrays(P, Q)
    out = ctypes.c_size_t()
    _check(_lib.kron_matmul_workspace_size(M, len(P), Pa, Qa, dtype_code(dtype, mode), ctypes.byref(out)),
           "kron_matmul_workspace_size")
    return int(out.value)


def plan_describe(M: int, P, Q, dtype, mode=None):
    """[(first factor (1-based), number fused, kernel family)] of the pass plan kron_matmul uses."""
    Pa, Qa = _shape_arrays(P, Q)
    cap = 64
    n = ctypes.c_int32()
    first = (ctypes.c_int32 * cap)()
    nf = (ctypes.c_int32 * cap)()
    kind = (ctypes.c_int32 * cap)()
    _check(_lib.kron_plan_describe(M, len(P), Pa, Qa, dtype_code(dtype, mode), cap, ctypes.byref(n), first, nf, kind),
           "kron_plan_describe")
    return [(first[i], nf[i], KIND_NAMES[kind[i]]) for i in range(n.value)]


def plan_kernels(M: int, P, Q, dtype, mode=None):
    """Kernel (family) name of every pass of the plan kron_matmul uses."""
    Pa, Qa = _shape_arrays(P, Q)
    out = []
    for i in range(len(plan_describe(M, P, Q, dtype, mode))):
        buf = ctypes.create_string_buffer(64)
        _check(_lib.kron_plan_kernel(M, len(P), Pa, Qa, dtype_code(dtype, mode), i, buf, 64), "kron_plan_kernel")
        out.append(buf.value.decode())
    return out


def plan_cost(M: int, P, Q, dtype, mode=None):
    """(algorithmic HBM bytes, FLOPs) of the plan."""
    Pa, Qa = _shape_arrays(P, Q)
    b, f = ctypes.c_double(), ctypes.c_double()
    _check(_lib.kron_plan_cost(M, len(P), Pa, Qa, dtype_code(dtype, mode), ctypes.byref(b), ctypes.byref(f)),
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


def matmul(X, Fs, out=None, stream=None, mode=None):
    """Y = X · (F^1 ⊗ … ⊗ F^N) on the current (or given) CUDA stream via kron_matmul().
    mode="3xtf32": float32 data in the separately reported 3xTF32 tensor-core mode."""
    import torch
    P, Q = _prep(X, Fs)
    L = 1
    for q in Q:
        L *= q
    if out is None:
        out = torch.empty((X.shape[0], L), dtype=X.dtype, device=X.device)
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    _check(_lib.kron_matmul(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(), dtype_code(X.dtype, mode),
                            _stream_ptr(stream)), "kron_matmul")
    return out


def matmul_host(X, Fs, out=None, chunk_rows: int = 0, stream=None, mode=None):
    """kron_matmul_host(): X, Fs and out are CPU tensors (pin_memory() for overlap); the library streams
    row chunks host -> device -> host with the copies overlapping the passes.  Asynchronous on
    `stream` (synchronise before reading `out`)."""
    import torch
    if X.dim() != 2 or X.is_cuda or not X.is_contiguous():
        raise ValueError("X must be a contiguous 2-D CPU tensor")
    P = [int(f.shape[0]) for f in Fs]
    Q = [int(f.shape[1]) for f in Fs]
    for f in Fs:
        if f.is_cuda or not f.is_contiguous() or f.dtype != X.dtype or f.dim() != 2:
            raise ValueError("factors must be contiguous 2-D CPU tensors of X's dtype")
    K = L = 1
    for p, q in zip(P, Q):
        K, L = K * p, L * q
    if X.shape[1] != K:
        raise ValueError(f"X has {X.shape[1]} columns, prod P = {K}")
    if out is None:
        out = torch.empty((X.shape[0], L), dtype=X.dtype, pin_memory=X.is_pinned())
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    _check(_lib.kron_matmul_host(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(),
                                 dtype_code(X.dtype, mode), chunk_rows, _stream_ptr(stream)), "kron_matmul_host")
    return out


def matmul_ws(X, Fs, out, workspace, stream=None, mode=None):
    """kron_matmul_ws(): caller-owned output and workspace (a uint8 CUDA tensor, or None if 0 bytes)."""
    P, Q = _prep(X, Fs)
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    wptr = workspace.data_ptr() if workspace is not None else None
    wbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(_lib.kron_matmul_ws(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(), dtype_code(X.dtype, mode),
                               wptr, wbytes, _stream_ptr(stream)), "kron_matmul_ws")
    return out


def matmul_ws_events(X, Fs, out, workspace, events, stream=None, mode=None):
    """kron_matmul_ws_events(): like matmul_ws, recording events[i] (raw cudaEvent_t handles) before
    pass i and events[npasses] after the last pass, for per-kernel timing."""
    P, Q = _prep(X, Fs)
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    Ev = (ctypes.c_void_p * len(events))(*[int(e) for e in events])
    wptr = workspace.data_ptr() if workspace is not None else None
    wbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(_lib.kron_matmul_ws_events(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(),
                                      dtype_code(X.dtype, mode), wptr, wbytes, Ev, len(events), _stream_ptr(stream)),
           "kron_matmul_ws_events")
    return out


def autotune(X, Fs, out=None, reps: int = 3, stream=None, mode=None):
    """kron_autotune(): time every candidate plan on these buffers, install the fastest for this
    (device, M, shapes, dtype).  Returns (Y, number of candidates, best ms)."""
    import torch
    P, Q = _prep(X, Fs)
    L = 1
    for q in Q:
        L *= q
    if out is None:
        out = torch.empty((X.shape[0], L), dtype=X.dtype, device=X.device)
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    n, ms = ctypes.c_int32(), ctypes.c_float()
    _check(_lib.kron_autotune(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(), dtype_code(X.dtype, mode),
                              reps, _stream_ptr(stream), ctypes.byref(n), ctypes.byref(ms)), "kron_autotune")
    return out, n.value, ms.value


def autotune_candidates(M: int, P, Q, dtype, mode=None) -> int:
    Pa, Qa = _shape_arrays(P, Q)
    n = ctypes.c_int32()
    _check(_lib.kron_autotune_candidates(M, len(P), Pa, Qa, dtype_code(dtype, mode), ctypes.byref(n)),
           "kron_autotune_candidates")
    return n.value


def plan_cache_clear() -> None:
    _check(_lib.kron_plan_cache_clear(), "kron_plan_cache_clear")


class Graph:
    """kron_graph_create(): the plan's launches for these exact tensors captured in a CUDA graph;
    launch() enqueues one Kron-Matmul at graph-replay cost (contents may change, storage may not)."""

    def __init__(self, X, Fs, out, workspace, mode=None):
        P, Q = _prep(X, Fs)
        Pa, Qa = _shape_arrays(P, Q)
        Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
        wptr = workspace.data_ptr() if workspace is not None else None
        wbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
        h = ctypes.c_void_p()
        _check(_lib.kron_graph_create(X.shape[0], len(P), Pa, Qa, X.data_ptr(), Fp, out.data_ptr(),
                                      dtype_code(X.dtype, mode), wptr, wbytes, ctypes.byref(h)), "kron_graph_create")
        self.handle = h.value
        self._keep = (X, list(Fs), out, workspace)  # the captured pointers must stay alive

    def launch(self, stream=None):
        _check(_lib.kron_graph_launch(self.handle, _stream_ptr(stream)), "kron_graph_launch")

    def close(self):
        if getattr(self, "handle", None):
            _lib.kron_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()


def raw_lib():
    return _lib


# ------------------------------------------------------------------ distributed (Algorithm 2)

_lib.kron_dist_nccl_unique_id.restype = ctypes.c_int
_lib.kron_dist_nccl_unique_id.argtypes = [ctypes.c_void_p]
_lib.kron_dist_ctx_create.restype = ctypes.c_int
_lib.kron_dist_ctx_create.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]
_lib.kron_dist_p2p_heap_bytes.restype = ctypes.c_int
_lib.kron_dist_p2p_heap_bytes.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]
_lib.kron_dist_p2p_reserve.restype = ctypes.c_int
_lib.kron_dist_p2p_reserve.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
_lib.kron_dist_p2p_connect.restype = ctypes.c_int
_lib.kron_dist_p2p_connect.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
_lib.kron_dist_p2p_timeouts.restype = ctypes.c_int
_lib.kron_dist_p2p_timeouts.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32)]
_lib.kron_dist_ctx_destroy.restype = ctypes.c_int
_lib.kron_dist_ctx_destroy.argtypes = [ctypes.c_void_p]
_lib.kron_dist_ctx_grid.restype = ctypes.c_int
_lib.kron_dist_ctx_grid.argtypes = [ctypes.c_void_p, _i32p, _i32p]
_lib.kron_dist_ctx_set.restype = ctypes.c_int
_lib.kron_dist_ctx_set.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
_lib.kron_dist_sync.restype = ctypes.c_int
_lib.kron_dist_sync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
_lib.kron_dist_round_layouts.restype = ctypes.c_int
_lib.kron_dist_round_layouts.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
_lib.kron_dist_round_info.restype = ctypes.c_int
_lib.kron_dist_round_info.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_int32, _i32p, _i32p, _i32p]
KRON_DIST_OPT_CHUNKS, KRON_DIST_OPT_FUSED_LAYOUT, KRON_DIST_OPT_P2P_PUSH = 1, 2, 3
_lib.kron_matmul_dist.restype = ctypes.c_int
_lib.kron_matmul_dist.argtypes = [ctypes.c_int64, ctypes.c_int32, _i32p, _i32p, ctypes.c_void_p, _vpp, ctypes.c_void_p,
                                  ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]


class DistContext:
    """kron_dist_ctx_t.  backend "nccl": one rank per GPU; the ncclUniqueId is created by rank 0 and
    broadcast over the torch ProcessGroup `pg` (plumbing only).  backend "virtual": all GM*GK ranks of the
    grid live in this process on the current GPU (exchange = device copies).  GM = GK = 0: the paper's
    grid rule.  Options (identical on every rank): `chunks` row chunks per round (NCCL /
    virtual: chunk c's all-to-all overlaps chunk c+1's passes), `fused` the fused send / receive layouts
    (False = separate pack and remap kernels), `push` the P2P backend's fused push rounds (None = the
    library default, fixed at creation)."""

    def __init__(self, backend="nccl", world_size=None, rank=None, GM=0, GK=0, pg=None, chunks=None, fused=None,
                 push=None):
        self.handle = ctypes.c_void_p()
        if backend == "nccl":
            import torch.distributed as dist
            world_size = dist.get_world_size(pg) if world_size is None else world_size
            rank = dist.get_rank(pg) if rank is None else rank
            uid = ctypes.create_string_buffer(128)
            if rank == 0:
                _check(_lib.kron_dist_nccl_unique_id(uid), "kron_dist_nccl_unique_id")
            obj = [bytes(uid.raw) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=pg)
            uid = ctypes.create_string_buffer(obj[0], 128)
            _check(_lib.kron_dist_ctx_create(0, uid, world_size, rank, GM, GK, ctypes.byref(self.handle)),
                   "kron_dist_ctx_create")
        elif backend == "p2p":
            # peer-memory exchange (backend 2): the symmetric heap is reserved lazily by matmul_dist,
            # collectively, with its CUDA IPC handles all-gathered over `pg` (plumbing only)
            import torch.distributed as dist
            world_size = dist.get_world_size(pg) if world_size is None else world_size
            rank = dist.get_rank(pg) if rank is None else rank
            _check(_lib.kron_dist_ctx_create(2, None, world_size, rank, GM, GK, ctypes.byref(self.handle)),
                   "kron_dist_ctx_create")
        elif backend == "virtual":
            if world_size is None:
                world_size = GM * GK
            _check(_lib.kron_dist_ctx_create(1, None, world_size, 0, GM, GK, ctypes.byref(self.handle)),
                   "kron_dist_ctx_create")
            rank = 0
        else:
            raise ValueError(backend)
        self.backend, self.rank, self.world_size = backend, rank, world_size
        self.pg, self.heap_bytes = pg, 0
        gm, gk = ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.kron_dist_ctx_grid(self.handle, ctypes.byref(gm), ctypes.byref(gk)), "kron_dist_ctx_grid")
        self.GM, self.GK = gm.value, gk.value
        for opt, val in ((KRON_DIST_OPT_CHUNKS, chunks), (KRON_DIST_OPT_FUSED_LAYOUT, fused),
                         (KRON_DIST_OPT_P2P_PUSH, push)):
            if val is not None:
                _check(_lib.kron_dist_ctx_set(self.handle, opt, int(val)), "kron_dist_ctx_set")

    def sync(self, stream=None, timeout_ms: int = 120000) -> None:
        """kron_dist_sync: wait for `stream`, polling NCCL's asynchronous errors (raises KronError with
        KRON_ERR_NCCL / KRON_ERR_CUDA on a failed or stuck collective or a P2P barrier that gave up)."""
        _check(_lib.kron_dist_sync(self.handle, _stream_ptr(stream), int(timeout_ms)), "kron_dist_sync")

    def round_info(self, M, P, Q, dtype):
        """[(fused_send, fused_recv)] per round for this context's grid (host only)."""
        Pa, Qa = _shape_arrays(P, Q)
        n = ctypes.c_int32()
        fs, fr = (ctypes.c_int32 * 64)(), (ctypes.c_int32 * 64)()
        _check(_lib.kron_dist_round_info(M, len(P), Pa, Qa, dtype_code(dtype), self.handle, 64, ctypes.byref(n),
                                         fs, fr), "kron_dist_round_info")
        return [(bool(fs[i]), bool(fr[i])) for i in range(n.value)]

    def round_layouts(self, M, P, Q, dtype):
        """Per round: the exchange layout of backends 0 / 1 — "plain", "direct-index" or "tile-major" (host only)."""
        Pa, Qa = _shape_arrays(P, Q)
        n = ctypes.c_int32()
        lay = (ctypes.c_int32 * 64)()
        _check(_lib.kron_dist_round_layouts(M, len(P), Pa, Qa, dtype_code(dtype), self.handle, 64, ctypes.byref(n), lay),
               "kron_dist_round_layouts")
        return [("plain", "direct-index", "tile-major")[lay[i]] for i in range(n.value)]

    def ensure_heap(self, nbytes: int) -> None:
        """P2P backend: (re)reserve the symmetric heap if it is smaller than `nbytes` and map the peers'
        heaps.  Collective: every rank calls it with the same size (matmul_dist does)."""
        if nbytes <= self.heap_bytes:
            return
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        dist.barrier(group=self.pg)  # nobody still reads the old heaps
        h = ctypes.create_string_buffer(64)
        _check(_lib.kron_dist_p2p_reserve(self.handle, nbytes, h), "kron_dist_p2p_reserve")
        allh = [None] * self.world_size
        dist.all_gather_object(allh, bytes(h.raw), group=self.pg)
        buf = ctypes.create_string_buffer(b"".join(allh), 64 * self.world_size)
        _check(_lib.kron_dist_p2p_connect(self.handle, buf), "kron_dist_p2p_connect")
        self.heap_bytes = nbytes

    def timeouts(self) -> int:
        """P2P backend: barrier waits that gave up (0 in a healthy run; synchronizes)."""
        c = ctypes.c_uint32()
        _check(_lib.kron_dist_p2p_timeouts(self.handle, ctypes.byref(c)), "kron_dist_p2p_timeouts")
        return c.value

    def coords(self, rank=None):
        r = self.rank if rank is None else rank
        return r // self.GK, r % self.GK

    def close(self):
        if self.handle:
            _lib.kron_dist_ctx_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def matmul_dist(M, X_local, Fs, ctx: DistContext, out=None, stream=None, check: bool = False):
    """kron_matmul_dist().  nccl / p2p backends: X_local is this rank's block X[gM rows, gK K-block]; returns
    Y_local = Y[gM rows, gK L-block].  virtual backend: X_local is a list of every rank's block (rank
    order gM*GK + gK); returns the list of Y_local blocks.  check=True waits for the result and raises on an
    asynchronous NCCL error or a P2P barrier timeout (ctx.sync)."""
    import torch
    if not Fs:
        raise ValueError("at least one factor")
    P = [int(f.shape[0]) for f in Fs]
    Q = [int(f.shape[1]) for f in Fs]
    K, L = 1, 1
    for p, q in zip(P, Q):
        K, L = K * p, L * q
    xs = list(X_local) if isinstance(X_local, (list, tuple)) else [X_local]
    nblk = ctx.GM * ctx.GK if ctx.backend == "virtual" else 1
    if len(xs) != nblk:
        raise ValueError(f"{ctx.backend} backend expects {nblk} X block(s), got {len(xs)}")
    if M % ctx.GM or K % ctx.GK or L % ctx.GK:
        raise ValueError(f"grid {ctx.GM}x{ctx.GK} does not divide M={M}, K={K}, L={L}")
    xshape, shape = (M // ctx.GM, K // ctx.GK), (M // ctx.GM, L // ctx.GK)
    dt, dev = xs[0].dtype, xs[0].device
    for x in xs:
        if not x.is_cuda or not x.is_contiguous() or x.dtype != dt or x.device != dev or tuple(x.shape) != xshape:
            raise ValueError(f"X blocks must be contiguous {dt} CUDA tensors of shape {xshape} on {dev}")
    for f in Fs:
        if not f.is_cuda or not f.is_contiguous() or f.dtype != dt or f.device != dev or f.dim() != 2:
            raise ValueError(f"factors must be contiguous 2-D {dt} CUDA tensors on {dev}")
    if out is None:
        outs = [torch.empty(shape, dtype=dt, device=dev) for _ in xs]
    else:
        outs = list(out) if isinstance(out, (list, tuple)) else [out]
        if len(outs) != len(xs):
            raise ValueError(f"expected {len(xs)} output block(s), got {len(outs)}")
        for y in outs:
            if not y.is_cuda or not y.is_contiguous() or y.dtype != dt or y.device != dev or tuple(y.shape) != shape:
                raise ValueError(f"output blocks must be contiguous {dt} CUDA tensors of shape {shape} on {dev}")
    Pa, Qa = _shape_arrays(P, Q)
    Fp = (ctypes.c_void_p * len(Fs))(*[f.data_ptr() for f in Fs])
    if ctx.backend == "p2p":
        need = ctypes.c_size_t()
        _check(_lib.kron_dist_p2p_heap_bytes(M, len(P), Pa, Qa, dtype_code(dt), ctx.GM, ctx.GK,
                                             ctypes.byref(need)), "kron_dist_p2p_heap_bytes")
        ctx.ensure_heap(need.value)
    if ctx.backend == "virtual":
        xp = (ctypes.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
        yp = (ctypes.c_void_p * len(outs))(*[y.data_ptr() for y in outs])
        xarg, yarg = ctypes.cast(xp, ctypes.c_void_p), ctypes.cast(yp, ctypes.c_void_p)
    else:
        xarg, yarg = xs[0].data_ptr(), outs[0].data_ptr()
    _check(_lib.kron_matmul_dist(M, len(P), Pa, Qa, xarg, Fp, yarg, dtype_code(dt), ctx.handle,
                                 _stream_ptr(stream)), "kron_matmul_dist")
    if check:
        ctx.sync(stream)
    return outs if isinstance(X_local, (list, tuple)) else outs[0]
