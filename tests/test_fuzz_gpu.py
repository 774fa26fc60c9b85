"""Seeded shape fuzz: the CUDA path (through the C-ABI) against the CPU oracle on random factor shapes.

Shapes are drawn so that every kernel family gets exercised by some of them — runs of equal square
factors (fused groups: factor pipeline, chunk pairs, the 16x16 cluster triple), large P (GEMM passes),
mixed / non-square / odd shapes (generic), M from 1 to a few tens (ragged row blocks) — with K*L bounded
so the oracle finishes in seconds.  Small-integer data: every partial sum is exact, so the comparison is
bit-exact whatever the summation order (parity bars).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _shapes(n=120, seed=2401):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        kind = rng.integers(0, 6)
        if kind == 4:      # fp32 16x16 runs long enough for the cluster triple (W >= 8 chunks of 4096)
            P = [16] * int(rng.integers(3, 6))
            if rng.integers(0, 2):
                P = [int(rng.choice([2, 4, 8]))] + P
            Q = list(P)
        elif kind == 5:    # fp64 chunk pairs on DMMA: 32x32 pairs, 64x32 GP pairs
            if rng.integers(0, 2):
                P, Q = [32] * int(rng.integers(2, 4)), None
                Q = list(P)
            else:
                P = [64] * int(rng.integers(2, 4))
                Q = [32] * len(P)
        elif kind == 0:    # run of equal square factors (fused groups)
            p = int(rng.choice([2, 4, 8, 16, 32]))
            N = int(rng.integers(2, 7))
            P = [p] * N
            Q = list(P)
        elif kind == 1:    # square runs behind / before an odd factor
            p = int(rng.choice([8, 16]))
            P = [p] * int(rng.integers(2, 5))
            x = int(rng.choice([2, 3, 5, 8]))
            P = [x] + P if rng.integers(0, 2) else P + [x]
            Q = list(P)
        elif kind == 2:    # large P / non-square GP-style factors
            P = [int(rng.choice([48, 64, 128])) for _ in range(int(rng.integers(1, 3)))]
            Q = [int(rng.choice([16, 32, 64])) for _ in P]
        else:              # anything small and mixed
            N = int(rng.integers(1, 5))
            P = [int(rng.integers(1, 9)) for _ in range(N)]
            Q = [int(rng.integers(1, 9)) for _ in range(N)]
        K, L = int(np.prod(P)), int(np.prod(Q))
        M = int(rng.integers(1, 40))
        if K * M > (1 << 23) or L * M > (1 << 23) or K > (1 << 21):
            M = max(1, (1 << 23) // max(K, L))
            if K > (1 << 21) or M < 1:
                continue
        dt = np.float64 if rng.integers(0, 2) else np.float32
        if kind == 4:
            dt = np.float32
        elif kind == 5:
            dt = np.float64
        out.append((M, P, Q, dt))
    return out


@pytest.mark.parametrize("M,P,Q,dt", _shapes() + _shapes(120, seed=10187) + _shapes(120, seed=2026))
def test_fuzz_bit_exact(cuda_device, M, P, Q, dt):
    import torch
    from paper_2401_10187_b200 import kron
    seed = synth.SEED_BASE + 7000 + M
    mode = "int" if dt == np.float64 else "int1"
    X = synth.matrix(M, int(np.prod(P)), seed, 0, mode, dt)
    Fs = synth.factors(P, Q, seed, mode, dt)
    Y = kron.matmul(torch.from_numpy(X).to(cuda_device), [torch.from_numpy(f).to(cuda_device) for f in Fs])
    torch.cuda.synchronize()
    ref = oracle.alg1(X, Fs).astype(dt)
    assert np.array_equal(Y.cpu().numpy(), ref), (M, P, Q, kron.plan_kernels(M, P, Q, np.dtype(dt).name))
