"""paper_2401_10187_b200 — B200-native (sm_100a) Kron-Matmul, the hot path of FastKron
(arxiv 2401.10187): ``Y = X · (F^1 ⊗ … ⊗ F^N)`` as fused, direct-index sliced multiplies.

All arithmetic runs in ``libkron.so`` (hand-written CUDA behind the C-ABI in ``include/kron.h``);
this package only marshals arguments.  PyTorch supplies device memory, streams and process groups.
There is no CPU fallback: if ``libkron.so`` is missing, importing :mod:`.kron` raises.
"""
from .kron import (KronError, dtype_code, matmul, matmul_ws, plan_cost, plan_describe, workspace_size,  # noqa: F401
                   lib_path)

__all__ = ["KronError", "dtype_code", "matmul", "matmul_ws", "plan_cost", "plan_describe", "workspace_size",
           "lib_path"]
