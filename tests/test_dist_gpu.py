"""GPU parity of the distributed path (Algorithm 2) through kron_matmul_dist.

Only one GPU is available per run, so the grid runs on the "virtual" backend: all GM*GK ranks in one
process on cuda:0, exchanging with device copies.  It executes the NCCL backend's code path — round
planner, row chunks, local fused / GEMM passes whose last pass writes the destination-major send buffer
(fused pack), the next round's first pass reading the receive buffer through the StoreGPUTile-ordered
tensor map (fused remap), the separate pack / StoreGPUTile kernels where a kernel has no such hook — with
the same buffers; only the all-to-all transport differs.  Every rank's Y_local is compared with the oracle's rows/columns block (rows are
independent, so no gather is needed): bit-exact on integer data, tolerance on random data.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kron(cuda_device):
    from paper_2401_10187_b200 import kron as k
    return k


GRIDS = [
    # (GM, GK, M, P, Q)
    (1, 2, 4, [16] * 5, [16] * 5),   # config E shapes, K split only (2 rounds: 3 + 2)
    (2, 2, 8, [16] * 5, [16] * 5),   # paper rule for 4 GPUs
    (4, 2, 8, [16] * 5, [16] * 5),   # paper rule for 8 GPUs
    (2, 1, 6, [8] * 6, [8] * 6),     # row-only: no exchange
    (1, 4, 2, [4] * 4, [4] * 4),     # Fig 8: {1,4}, K = 256, Local = 2
    (2, 4, 4, [8] * 4, [8] * 4),
    (1, 8, 3, [8] * 5, [8] * 5),
    (2, 2, 4, [8, 4, 4], [4, 8, 4]),  # mixed, non-square
    (1, 2, 2, [64, 64], [32, 32]),    # large P, GEMM passes per round
    (1, 2, 3, [2, 16, 16, 16, 8, 8], [2, 16, 16, 16, 8, 8]),  # v9 ends a round with rho = 1 (no float4 push)
    (1, 2, 3, [2, 16, 16, 8, 8, 4, 4], [2, 16, 16, 8, 8, 4, 4]),  # 3-pass round ending in a v6 pair
    (1, 2, 5, [32] * 4, [32] * 4),    # C32 shapes: v6 P = 32 pairs with the fused send / receive layout
    (2, 2, 2, [64] * 4, [64] * 4),    # Fig 11 weak-scaling workload shape (P = 64, N = 4), K = 2^24
]
# (chunks, fused): the default (2 row chunks, fused layouts), the unfused kernels, ragged chunks
MODES = [(2, True), (1, False), (3, True)]


def run_virtual(kron, dev, GM, GK, M, P, Q, dt, mode, chunks=2, fused=True):
    import torch
    seed = synth.SEED_BASE + 300
    K = int(np.prod(P))
    X = synth.matrix(M, K, seed, 0, mode, dt)
    Fs = synth.factors(P, Q, seed, mode, dt)
    ctx = kron.DistContext("virtual", GM=GM, GK=GK, chunks=chunks, fused=fused)
    assert (ctx.GM, ctx.GK) == (GM, GK)
    Ml, Kl = M // GM, K // GK
    blocks = []
    for r in range(GM * GK):
        gm, gk = ctx.coords(r)
        blocks.append(torch.from_numpy(np.ascontiguousarray(X[gm * Ml:(gm + 1) * Ml, gk * Kl:(gk + 1) * Kl])).to(dev))
    Fd = [torch.from_numpy(f).to(dev) for f in Fs]
    Ys = kron.matmul_dist(M, blocks, Fd, ctx, check=True)
    torch.cuda.synchronize()
    ref = oracle.alg1(X, Fs)
    L = ref.shape[1]
    Ll = L // GK
    out = []
    for r, y in enumerate(Ys):
        gm, gk = ctx.coords(r)
        out.append((y.cpu().numpy(), ref[gm * Ml:(gm + 1) * Ml, gk * Ll:(gk + 1) * Ll]))
    ctx.close()
    return out


@pytest.mark.parametrize("chunks,fused", MODES)
@pytest.mark.parametrize("GM,GK,M,P,Q", GRIDS)
def test_dist_virtual_bit_exact(kron, cuda_device, GM, GK, M, P, Q, chunks, fused):
    for y, ref in run_virtual(kron, cuda_device, GM, GK, M, P, Q, np.float64, "int", chunks, fused):
        assert np.array_equal(y, ref)


@pytest.mark.parametrize("chunks,fused", MODES)
@pytest.mark.parametrize("GM,GK,M,P,Q", GRIDS[:4] + GRIDS[-3:])
def test_dist_virtual_random_fp32(kron, cuda_device, GM, GK, M, P, Q, chunks, fused):
    for y, ref in run_virtual(kron, cuda_device, GM, GK, M, P, Q, np.float32, "urand", chunks, fused):
        assert float(np.max(np.abs(y - ref) / np.abs(ref))) <= 1e-5


def test_dist_config_e_fused_layout(kron, cuda_device):
    # config E's rounds on the paper-rule grid for 8 GPUs {4,2}: round 1 (3 factors, v9 cluster
    # kernel) writes the send buffer from its store warps, round 2 (2 factors, v6) reads the receive buffer
    # through the remapped tensor map and writes its own send buffer; 16 rows per rank, 3 row chunks
    ctx = kron.DistContext("virtual", GM=4, GK=2, chunks=3)
    assert ctx.round_info(64, [16] * 5, [16] * 5, "float32") == [(True, False), (True, True)]
    ctx.close()
    for y, ref in run_virtual(kron, cuda_device, 4, 2, 64, [16] * 5, [16] * 5, np.float32, "int1", 3, True):
        assert np.array_equal(y, ref.astype(np.float32))


def test_dist_layout_errors(kron, cuda_device):
    import torch
    ctx = kron.DistContext("virtual", GM=4, GK=2)
    X = [torch.zeros((1, 8 ** 3 // 2), device=cuda_device) for _ in range(8)]
    Fs = [torch.eye(8, device=cuda_device)] * 3
    with pytest.raises(ValueError, match="does not divide"):
        kron.matmul_dist(6, X, Fs, ctx)  # GM = 4 does not divide M = 6 (the binding checks before the C call)
    with pytest.raises(ValueError, match="X block"):
        kron.matmul_dist(8, X[:7], Fs, ctx)  # the virtual backend needs GM*GK blocks
    with pytest.raises(ValueError, match="X blocks"):
        kron.matmul_dist(8, X, Fs, ctx)  # blocks of 1 row, M/GM = 2 expected
    ctx.close()
    with pytest.raises(kron.KronError):
        kron.DistContext("virtual", world_size=6)  # grid rule does not yield 6 GPUs (G14)


@pytest.mark.parametrize("GM,GK,M", [(1, 2, 4), (2, 4, 8), (1, 8, 3)])
def test_dist_config_e_tile_major_rounds(kron, cuda_device, GM, GK, M):
    # v11 through the exchange: round 1's triple writes the send blocks tile-major, round 2's pair reads the
    # receive blocks through a 4-D map (a source-rank dimension) and pushes into the final send blocks — the
    # kernels must be the tile-major ones and every rank's block bit-exact on integer data
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res = run_virtual(kron, cuda_device, GM, GK, M, [16] * 5, [16] * 5, np.float32, "int1", 2, True)
        torch.cuda.synchronize()
    names = " ".join(e.name for e in prof.events())
    assert "kron_tri_tm_kernel" in names and "kron_pair_tm_kernel" in names
    assert "gemm3c" not in names and "store_gpu_tile" in names  # only the final remap into Y_local
    for y, ref in res:
        assert np.array_equal(y, ref.astype(np.float32))
