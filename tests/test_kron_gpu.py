"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Bars: bit-exact on small-integer data (fp64 {-2..2}, fp32 {-1,0,1}: every partial
sum is an exact integer, so any summation order gives identical bits); max relative error <= 1e-5
(fp32) / 1e-12 (fp64) on U[0,1) data (positive: no cancellation); componentwise-normwise error on
signed data.  Sizes span several tiles plus ragged row blocks; full BASELINE sizes are checked on
sampled rows (the oracle computes rows independently).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}


@pytest.fixture(scope="module")
def kron(cuda_device):
    from paper_2401_10187_b200 import kron as k
    return k


def to_dev(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def run(kron, X, Fs, dev):
    import torch
    Y = kron.matmul(to_dev(X, dev), [to_dev(f, dev) for f in Fs])
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def case(M, P, Q, dt, mode, seed_off=0):
    seed = synth.SEED_BASE + 1000 + seed_off
    X = synth.matrix(M, int(np.prod(P)), seed, 0, mode, dt)
    Fs = synth.factors(P, Q, seed, mode, dt)
    return X, Fs


def rel_err(Y, ref):
    return float(np.max(np.abs(Y.astype(np.float64) - ref) / np.abs(ref)))


SMALL = [
    # (M, P, Q) — covers every kernel family and the degenerate cases
    (16, [4, 4], [4, 4]),                 # config A (generic)
    (17, [4] * 4, [4] * 4),               # fused P=4, ragged row block (tileM rows)
    (33, [8] * 4, [8] * 4),               # fused P=8 (3,1)
    (5, [8] * 6, [8] * 6),                # config B shape, small M (two separate passes)
    (3, [16] * 4, [16] * 4),              # fused P=16 (2,2)
    (3, [16] * 5, [16] * 5),              # config E shape: v11 triple -> pair with the tile-major hand-off
    (1, [16] * 5, [16] * 5),              # v11 hand-off, one row (a single triple tile per 4 chunks)
    (7, [16] * 5, [16] * 5),              # v11 hand-off, ragged row count over the persistent grid
    (5, [8, 16, 16, 16], [8, 16, 16, 16]),  # v9 triple (W = 8 chunks) behind a P=8 factor
    (2, [32] * 3, [32] * 3),              # fused P=32 (2,1)
    (9, [2] * 10, [2] * 10),              # fused P=2 deep groups
    (1, [8] * 5, [8] * 5),                # single row
    (7, [3, 5, 2], [2, 4, 3]),            # odd non-square -> generic
    (4, [8, 2], [2, 8]),                  # mixed widths (G2)
    (6, [5, 8, 8, 8], [5, 8, 8, 8]),      # odd leading factor + fused 8-run
    (3, [64, 64], [32, 32]),              # non-square large P (fp64: fused 64x32 pair on DMMA)
    (4, [64] * 3, [32] * 3),              # config D2 shape, small M (fused pair + single factor)
    (3, [2, 64, 64], [2, 32, 32]),        # fused 64x32 pair behind a tiny leading factor
    (2, [128, 16], [128, 16]),            # large P then small
    (4, [7], [9]),                        # N = 1: plain GEMM
    (3, [1, 4, 1], [2, 4, 1]),            # P_i or Q_i = 1
    # fp32 large-P passes on kron_sgemm_kernel (the three column-tile instances, ragged tiles, idle warps)
    (5, [64] * 3, [64] * 3),              # Fig 11 W64 shape (QT 16 x QR 4)
    (3, [128, 128], [128, 128]),          # W128 shape (QT 16 x QR 8), 384 slices = 1.5 tiles
    (7, [48, 64], [48, 16]),              # P = 48 (zero-padded 32-p chunk), Q = 48 / 16 (idle column ranges)
    (2, [96, 64], [80, 32]),              # Q = 80 in a 128-column tile, Q = 32 (QT 8 x QR 4)
    (5, [64, 3], [64, 3]),                # S = 3 slices per row: a warp's 32 slices span 11 rows
]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("M,P,Q", SMALL)
def test_bit_exact_integer(kron, cuda_device, M, P, Q, dt):
    mode = "int1" if dt == np.float32 else "int"
    X, Fs = case(M, P, Q, dt, mode)
    ref = oracle.alg1(X, Fs)
    assert np.max(np.abs(ref)) < (2 ** 24 if dt == np.float32 else 2 ** 53)
    Y = run(kron, X, Fs, cuda_device)
    assert Y.dtype == dt
    assert np.array_equal(Y, ref.astype(dt)), f"max |diff| {np.max(np.abs(Y - ref))}"


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("M,P,Q", SMALL)
def test_random_relative_error(kron, cuda_device, M, P, Q, dt):
    X, Fs = case(M, P, Q, dt, "urand", 1)
    ref = oracle.alg1(X, Fs)
    Y = run(kron, X, Fs, cuda_device)
    assert rel_err(Y, ref) <= TOL[dt]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_signed_componentwise(kron, cuda_device, dt):
    M, P = 11, [8] * 5
    X, Fs = case(M, P, P, dt, "srand", 2)
    ref = oracle.alg1(X, Fs)
    den = oracle.alg1(np.abs(X), [np.abs(f) for f in Fs])  # (|X| . (x)|F|)
    Y = run(kron, X, Fs, cuda_device)
    assert float(np.max(np.abs(Y - ref) / den)) <= TOL[dt]


def test_identity_and_permutation_factors(kron, cuda_device):
    rng = np.random.default_rng(3)
    P = [8, 8, 8, 8]
    X = synth.matrix(19, 8 ** 4, synth.SEED_BASE, 0, "urand", np.float32)
    Y = run(kron, X, [np.eye(8, dtype=np.float32)] * 4, cuda_device)
    assert np.array_equal(Y, X)
    perms = [rng.permutation(8) for _ in P]
    Fs = [np.eye(8, dtype=np.float32)[p] for p in perms]
    Y = run(kron, X, Fs, cuda_device)
    assert np.array_equal(Y, oracle.alg1(X, Fs).astype(np.float32))  # a pure column permutation


def test_m_zero_and_empty(kron, cuda_device):
    import torch
    X = torch.empty((0, 64), dtype=torch.float32, device=cuda_device)
    F = [torch.eye(8, device=cuda_device)] * 2
    Y = kron.matmul(X, F)
    assert Y.shape == (0, 64)


def test_workspace_variant_and_stream(kron, cuda_device):
    import torch
    X, Fs = case(64, [8] * 6, [8] * 6, np.float32, "urand", 3)
    Xd, Fd = to_dev(X, cuda_device), [to_dev(f, cuda_device) for f in Fs]
    ws = torch.empty(kron.workspace_size(64, [8] * 6, [8] * 6, torch.float32), dtype=torch.uint8, device=cuda_device)
    out = torch.empty((64, 8 ** 6), dtype=torch.float32, device=cuda_device)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        kron.matmul_ws(Xd, Fd, out, ws)
    s.synchronize()
    assert rel_err(out.cpu().numpy(), oracle.alg1(X, Fs)) <= 1e-5
    with pytest.raises(kron.KronError):
        kron.matmul_ws(Xd, Fd, out, ws[:10])  # workspace too small -> KRON_ERR_SHAPE, nothing enqueued


# ------------------------------------------------------------------ full BASELINE sizes, sampled rows

FULL = [
    ("B", 1, 1024, [8] * 6, [8] * 6, np.float32),
    ("C32", 2, 1024, [32] * 4, [32] * 4, np.float32),
    ("C64", 2, 1024, [32] * 4, [32] * 4, np.float64),
    ("D1", 3, 320, [128] * 3, [128] * 3, np.float64),
    ("D2", 4, 320, [64] * 3, [32] * 3, np.float64),
    ("E", 5, 4096, [16] * 5, [16] * 5, np.float32),
]


@pytest.mark.slow
@pytest.mark.parametrize("name,cfg,M,P,Q,dt", FULL)
def test_full_size_sampled_rows(kron, cuda_device, name, cfg, M, P, Q, dt):
    import torch
    seed = synth.SEED_BASE + cfg
    K, L = int(np.prod(P)), int(np.prod(Q))
    tdt = torch.float32 if dt == np.float32 else torch.float64
    X = torch.empty((M, K), dtype=tdt, device=cuda_device)
    synth.fill_device(X.data_ptr(), M, K, seed, 0, "urand", dt)
    Fs_h = synth.factors(P, Q, seed, "urand", dt)
    Y = kron.matmul(X, [to_dev(f, cuda_device) for f in Fs_h])
    rows = synth.row_subset(M, extra=12)
    Ys = Y[torch.from_numpy(rows).to(cuda_device)].cpu().numpy()
    del X, Y
    torch.cuda.empty_cache()
    ref = oracle.alg1(synth.rows_of(rows, K, seed, 0, "urand"), Fs_h)
    assert rel_err(Ys, ref) <= TOL[dt]


@pytest.mark.parametrize("M,P,Q,dt", [
    (40, [8] * 6, [8] * 6, np.float32),
    (24, [32] * 4, [32] * 4, np.float64),
    (20, [16] * 5, [16] * 5, np.float32),
    (9, [64] * 3, [32] * 3, np.float64),
])
def test_autotuned_plan_parity(kron, cuda_device, M, P, Q, dt):
    # the autotuner times every candidate on the caller's buffers and installs the
    # fastest; its output and every later call through the installed plan stay bit-exact
    mode = "int1" if dt == np.float32 else "int"
    X, Fs = case(M, P, Q, dt, mode, 7)
    ref = oracle.alg1(X, Fs).astype(dt)
    Xd, Fd = to_dev(X, cuda_device), [to_dev(f, cuda_device) for f in Fs]
    Y, n, ms = kron.autotune(Xd, Fd, reps=2)
    assert n >= 1 and ms > 0
    assert np.array_equal(Y.cpu().numpy(), ref)
    assert np.array_equal(run(kron, X, Fs, cuda_device), ref)
    kron.plan_cache_clear()


# ------------------------------------------------------------------ fused chains of any square P (NEXT-3)

CHAIN = [
    (9, [3] * 7, [3] * 7),            # Table 4 #17 shape (3^7): one pass of seven fused factors, whole-row tile
    (5, [6] * 7, [6] * 7),            # Table 4 #19 shape (6^7): passes of 4 + 3 fused factors (even chunk, padded)
    (3, [5] * 4, [5] * 4),
    (4, [7] * 3 + [2], [7] * 3 + [2]),  # chain behind a single 2x2 factor
    (6, [12] * 3, [12] * 3),
    (2, [2] * 3 + [3] * 4, [2] * 3 + [3] * 4),  # mixed runs: fused power-of-2 and chain passes
]


@pytest.mark.parametrize("M,P,Q", CHAIN)
def test_chain_parity(kron, cuda_device, M, P, Q):
    import torch
    assert "kron_chain_kernel" in kron.plan_kernels(M, P, Q, "float32")
    for dt, data, seed_off in ((np.float32, "int1", 21), (np.float32, "urand", 22), (np.float64, "int", 23),
                               (np.float64, "urand", 24)):
        X, Fs = case(M, P, Q, dt, data, seed_off)
        ref = oracle.alg1(X, Fs)
        Y = kron.matmul(to_dev(X, cuda_device), [to_dev(f, cuda_device) for f in Fs])
        torch.cuda.synchronize()
        Y = Y.cpu().numpy()
        if data.startswith("int"):
            assert np.array_equal(Y, ref.astype(dt))
        else:
            assert rel_err(Y, ref) <= TOL[dt]


# ------------------------------------------------------------------ tensor-core modes (NEXT-4, tcgen05)

TC = [
    (40, [32] * 4, [32] * 4),         # two P = 32 pairs on the tcgen05 kernel (2 M-tiles per 8-chunk tile)
    (9, [32] * 3, [32] * 3),          # pair + single factor (CUDA cores)
    (3, [16, 32, 32], [16, 32, 32]),
    (5, [16] * 4, [16] * 4),          # P = 16 pairs (64B-swizzled K-major operand, 16-chunk tiles)
    (3, [16] * 5, [16] * 5),          # config E shape: CUDA-core triple + tensor-core pair
    (17, [8, 16, 16], [8, 16, 16]),   # rows shorter than a tensor-core tile: CUDA-core fallback
    (7, [32, 16, 16], [32, 16, 16]),  # pair behind a wider factor, odd M
]
# TF32 mode: positive U[0,1) data, products of operands with 10 explicit mantissa bits (truncated or
# rounded by the tensor core) through two contractions: relative error <= ~2 * 2 * 2^-10 ~ 4e-3; gate 5e-3
TF32_TOL = 5e-3


@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("M,P,Q", TC)
def test_tensor_core_mode_parity(kron, cuda_device, M, P, Q, mode):
    # small integers are exact in TF32 (lo = 0) and every partial sum is an exact fp32 integer -> bit exact in
    # both modes; U[0,1) data: 3xTF32 within the fp32 bar (~22-bit products), TF32 within TF32_TOL
    import torch
    for data, seed_off in (("int1", 11), ("urand", 12)):
        X, Fs = case(M, P, Q, np.float32, data, seed_off)
        ref = oracle.alg1(X, Fs)
        Y = kron.matmul(to_dev(X, cuda_device), [to_dev(f, cuda_device) for f in Fs], mode=mode)
        torch.cuda.synchronize()
        Y = Y.cpu().numpy()
        if data == "int1":
            assert np.array_equal(Y, ref.astype(np.float32))
        else:
            assert rel_err(Y, ref) <= (TOL[np.float32] if mode == "3xtf32" else TF32_TOL)
    R = 8 if P[-1] == 32 else 16  # chunks per tensor-core tile
    if P[-1] in (16, 32) and P[-2] == P[-1] and int(np.prod(P)) % (R * P[-1] ** 2) == 0:
        assert "kron_tc_pair_kernel" in kron.plan_kernels(M, P, Q, "float32", mode)


@pytest.mark.parametrize("M,P,Q", TC[:3])
def test_tf32x3_mma_sync_fallback(kron, cuda_device, M, P, Q):
    # round 1's mma.sync 3xTF32 kernel (P = 32 pairs) stays selectable by the autotuner when the tcgen05 kernel
    # is masked out (KRON_KINDS_MASK without bit 13); fresh process because plans are cached
    import os
    import subprocess
    import sys
    code = f"""
import numpy as np, torch, oracle, synth
from paper_2401_10187_b200 import kron
M, P, Q = {M}, {P}, {Q}
X = synth.matrix(M, int(np.prod(P)), synth.SEED_BASE + 12, 0, 'urand', np.float32)
Fs = synth.factors(P, Q, synth.SEED_BASE + 12, 'urand', np.float32)
Y = kron.matmul(torch.from_numpy(X).cuda(), [torch.from_numpy(f).cuda() for f in Fs], mode='3xtf32').cpu().numpy()
ref = oracle.alg1(X, Fs)
assert float(np.max(np.abs(Y - ref) / np.abs(ref))) <= 1e-5
assert 'kron_tc_pair_kernel' not in kron.plan_kernels(M, P, Q, 'float32', '3xtf32')
print('ok', kron.plan_kernels(M, P, Q, 'float32', '3xtf32'))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root,
                         env={**os.environ, "KRON_KINDS_MASK": "1FFF", "PYTHONPATH": root})
    assert "ok" in res.stdout, res.stdout + res.stderr


@pytest.mark.slow
def test_tf32x3_full_size_sampled_rows(kron, cuda_device):
    import torch
    M, P, seed = 1024, [32] * 4, synth.SEED_BASE + 2
    K = 32 ** 4
    X = torch.empty((M, K), dtype=torch.float32, device=cuda_device)
    synth.fill_device(X.data_ptr(), M, K, seed, 0, "urand", np.float32)
    Fs_h = synth.factors(P, P, seed, "urand", np.float32)
    rows = synth.row_subset(M, extra=12)
    ref = oracle.alg1(synth.rows_of(rows, K, seed, 0, "urand"), Fs_h)
    for mode, tol in (("3xtf32", TOL[np.float32]), ("tf32", TF32_TOL)):
        Y = kron.matmul(X, [to_dev(f, cuda_device) for f in Fs_h], mode=mode)
        Ys = Y[torch.from_numpy(rows).to(cuda_device)].cpu().numpy()
        del Y
        assert rel_err(Ys, ref) <= tol


@pytest.mark.parametrize("M,P,Q,dt", [(20, [2] * 7, [2] * 7, np.float32), (16, [8] * 3, [8] * 3, np.float64),
                                      (40, [32] * 4, [32] * 4, np.float32), (4, [64] * 3, [32] * 3, np.float64)])
def test_graph_replay(kron, cuda_device, M, P, Q, dt):
    # kron_graph_*: the captured plan replays bit-identically, and reads the buffers' current contents
    import torch
    X, Fs = case(M, P, Q, dt, "urand", 21)
    Xd, Fd = to_dev(X, cuda_device), [to_dev(f, cuda_device) for f in Fs]
    tdt = Xd.dtype
    ws = torch.empty(max(kron.workspace_size(M, P, Q, tdt), 1), dtype=torch.uint8, device=cuda_device)
    Y1 = torch.empty((M, int(np.prod(Q))), dtype=tdt, device=cuda_device)
    Y2 = torch.empty_like(Y1)
    kron.matmul_ws(Xd, Fd, Y1, ws)
    g = kron.Graph(Xd, Fd, Y2, ws)
    g.launch()
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    X2, _ = case(M, P, Q, dt, "int" if dt == np.float64 else "int1", 22)
    Xd.copy_(torch.from_numpy(X2))
    for _ in range(3):
        g.launch()
    torch.cuda.synchronize()
    g.close()
    # integer X with U[0,1) factors is not exact; compare against the direct call on the new data
    Y3 = torch.empty_like(Y1)
    kron.matmul_ws(Xd, Fd, Y3, ws)
    torch.cuda.synchronize()
    assert torch.equal(Y2, Y3)
    ref = oracle.alg1(X2, Fs)
    den = oracle.alg1(np.abs(X2), [np.abs(f) for f in Fs])
    assert float(np.max(np.abs(Y2.cpu().numpy() - ref) / np.maximum(den, 1e-300))) <= TOL[dt]


@pytest.mark.parametrize("M,P,Q,dt,chunk", [(37, [8] * 4, [8] * 4, np.float32, 8), (10, [32] * 3, [32] * 3, np.float64, 3),
                                            (9, [64] * 3, [32] * 3, np.float64, 4), (5, [3, 5], [4, 2], np.float32, 0)])
def test_host_path(kron, cuda_device, M, P, Q, dt, chunk):
    # kron_matmul_host: host buffers, row chunks (with a ragged tail) pipelined through two device slots
    import torch
    mode = "int1" if dt == np.float32 else "int"
    X, Fs = case(M, P, Q, dt, mode, 31)
    Xh = torch.from_numpy(X).pin_memory()
    Fh = [torch.from_numpy(f).pin_memory() for f in Fs]
    Y = kron.matmul_host(Xh, Fh, chunk_rows=chunk)
    torch.cuda.synchronize()
    assert np.array_equal(Y.numpy(), oracle.alg1(X, Fs).astype(dt))


# ------------------------------------------------------------------ v11 tile-major hand-off (config E plans)

_NOHO = """
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2401_10187_b200 import kron
d = np.load(sys.argv[1])
X = torch.from_numpy(d["X"]).cuda()
Fs = [torch.from_numpy(d["F%d" % i]).cuda() for i in range(5)]
assert kron.plan_kernels(X.shape[0], [16] * 5, [16] * 5, torch.float32) == ["kron_fused_gemm3c_kernel",
                                                                          "kron_fused_gemm2ws_kernel"]
np.save(sys.argv[2], kron.matmul(X, Fs).cpu().numpy())
"""


@pytest.mark.parametrize("M", [2, 37])
def test_handoff_bit_identical_to_direct_index_plan(kron, cuda_device, tmp_path, M):
    # the hand-off changes only the intermediate's element order (same products, same summation order), so Y
    # equals the v10 direct-index plan's bit for bit on random data; the v10 plan runs in a child process with
    # KRON_NO_HANDOFF=1 (read once per process)
    import os
    import subprocess
    import sys
    X, Fs = case(M, [16] * 5, [16] * 5, np.float32, "srand", 9)
    assert kron.plan_kernels(M, [16] * 5, [16] * 5, "float32") == ["kron_tri_tm_kernel", "kron_pair_tm_kernel"]
    Y = run(kron, X, Fs, cuda_device)
    np.savez(tmp_path / "in.npz", X=X, **{"F%d" % i: f for i, f in enumerate(Fs)})
    env = dict(os.environ, KRON_NO_HANDOFF="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", _NOHO, str(tmp_path / "in.npz"), str(tmp_path / "y.npy")], cwd=root,
                   env=env, check=True, timeout=600)
    Y10 = np.load(tmp_path / "y.npy")
    assert np.array_equal(Y.view(np.uint32), Y10.view(np.uint32))
    den = oracle.alg1(np.abs(X), [np.abs(f) for f in Fs])
    assert float(np.max(np.abs(Y - oracle.alg1(X, Fs)) / den)) <= TOL[np.float32]
