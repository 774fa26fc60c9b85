"""paper_2401_10187_b200 — B200-native (sm_100a) Kron-Matmul, the hot path of FastKron
(arxiv 2401.10187): ``Y = X · (F^1 ⊗ … ⊗ F^N)`` as fused, direct-index sliced multiplies.

All arithmetic runs in ``libkron.so`` (hand-written CUDA behind the C-ABI in ``include/kron.h``);
this package only marshals arguments.  PyTorch supplies device memory, streams and process groups.
There is no CPU fallback: if ``libkron.so`` is missing, the first use of the API raises ImportError.
(The binding is imported lazily so that ``paper_2401_10187_b200.build`` can run before the library
exists.)
"""
_API = ("KronError", "dtype_code", "matmul", "matmul_ws", "matmul_ws_events", "plan_cost", "plan_describe",
        "workspace_size", "lib_path", "dist_plan", "grid_rule", "DistContext", "matmul_dist")


def __getattr__(name):
    if name in _API:
        from . import kron
        return getattr(kron, name)
    raise AttributeError(name)


__all__ = list(_API)
