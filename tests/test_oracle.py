"""Pins for the CPU oracle (oracle/), all CPU-only (-m "not gpu").

Every oracle function is checked against something other than itself: values the paper prints
(tests/golden/*, each citing PAPER.md), a library routine (np.kron, np.matmul), an independent
algorithm written here from the paper (the shuffle algorithm), closed forms and
identities (identity / permutation / diagonal / one-hot / rank-1 / mixed-product / linearity).
Shapes include non-square, mixed and degenerate (P or Q = 1) factors so that a transposed
operand, a wrong digit order or a dropped term fails at least one test.
"""
import functools
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def np_kron(Fs):
    return functools.reduce(np.kron, Fs)


def int_factors(P, Q, seed, lo=-2, hi=3):
    rng = np.random.default_rng(seed)
    return [rng.integers(lo, hi, size=(p, q)).astype(np.float64) for p, q in zip(P, Q)]


def shuffle_algorithm(X, Fs):
    """O4: the shuffle algorithm, an independent route to Kron-Matmul.

    For i = N..1: reshape to (M*K/P) x P, matmul with F^i, reshape M x (K/P) x Q, transpose the
    last two dims, flatten to M x (Q*K/P).
    """
    Y = np.asarray(X, dtype=np.float64)
    M = Y.shape[0]
    for F in reversed(Fs):
        P, Q = F.shape
        K = Y.shape[1]
        Z = Y.reshape(M * (K // P), P) @ F          # step (a)
        Z = Z.reshape(M, K // P, Q).transpose(0, 2, 1)  # step (b)
        Y = Z.reshape(M, Q * (K // P))               # step (c)
    return Y


SHAPES = [
    ([2], [3]),
    ([3], [2]),
    ([2, 2], [2, 2]),
    ([4, 4], [4, 4]),
    ([2, 3], [3, 2]),
    ([8, 2], [2, 8]),
    ([3, 1, 2], [1, 4, 2]),
    ([1, 5], [2, 1]),
    ([2, 3, 4], [4, 3, 2]),
    ([5, 3], [3, 6]),
    ([2, 2, 2, 2], [3, 1, 2, 2]),
]


# ------------------------------------------------------------------ O1: definition


@pytest.mark.parametrize("P,Q", SHAPES)
def test_kron_product_matches_np_kron(P, Q):
    Fs = int_factors(P, Q, seed=sum(P) * 31 + sum(Q))
    G = oracle.kron_product(Fs)
    assert G.shape == (int(np.prod(P)), int(np.prod(Q)))
    assert np.array_equal(G, np_kron(Fs))  # integer data: exact


def test_kron_product_block_definition():
    # block (i,j) of F1 (x) F2 is f1_ij * F2 (F1 most significant).
    F1 = np.array([[1.0, 2.0], [3.0, 4.0]])
    F2 = np.array([[0.0, 1.0], [1.0, 0.0]])
    G = oracle.kron_product([F1, F2])
    for i in range(2):
        for j in range(2):
            assert np.array_equal(G[2 * i:2 * i + 2, 2 * j:2 * j + 2], F1[i, j] * F2)


@pytest.mark.parametrize("P,Q", SHAPES)
def test_naive_equals_dense_matmul(P, Q):
    Fs = int_factors(P, Q, seed=7 + len(P))
    X = np.random.default_rng(3).integers(-2, 3, size=(5, int(np.prod(P)))).astype(np.float64)
    assert np.array_equal(oracle.naive(X, Fs), X @ np_kron(Fs))


# ------------------------------------------------------------------ worked example


def test_fig2_worked_example():
    rows = golden_rows("fig2_sliced_multiply.txt")
    x = np.array([[float(v) for v in rows[0]]])
    F = np.array([[float(v) for v in rows[1]], [float(v) for v in rows[2]]])
    expect = np.array([float(v) for v in rows[3]])
    got = oracle.sliced_multiply(x, F)[0]
    assert np.array_equal(got, expect)


def test_fig2_symbolic_layout():
    # first intermediate row = [x11 f11 + x12 f21, x13 f11 + x14 f21, x11 f12 + x12 f22, x13 f12 + x14 f22]
    rng = np.random.default_rng(11)
    X = rng.integers(-9, 10, size=(2, 4)).astype(np.float64)
    F2 = rng.integers(-9, 10, size=(2, 2)).astype(np.float64)
    T = oracle.sliced_multiply(X, F2)
    for m in range(2):
        x = X[m]
        expect = [x[0] * F2[0, 0] + x[1] * F2[1, 0], x[2] * F2[0, 0] + x[3] * F2[1, 0],
                  x[0] * F2[0, 1] + x[1] * F2[1, 1], x[2] * F2[0, 1] + x[3] * F2[1, 1]]
        assert np.array_equal(T[m], expect)


# ------------------------------------------------------------------ O2: Algorithm 1


@pytest.mark.parametrize("P,Q", SHAPES)
def test_alg1_equals_bruteforce_integer(P, Q):
    Fs = int_factors(P, Q, seed=101 + sum(P))
    X = np.random.default_rng(5).integers(-2, 3, size=(7, int(np.prod(P)))).astype(np.float64)
    assert np.array_equal(oracle.alg1(X, Fs), oracle.naive(X, Fs))
    assert np.array_equal(oracle.alg1(X, Fs), X @ np_kron(Fs))


@pytest.mark.parametrize("P,Q", SHAPES)
def test_alg1_equals_shuffle_random(P, Q):
    rng = np.random.default_rng(17)
    Fs = [rng.standard_normal((p, q)) for p, q in zip(P, Q)]
    X = rng.standard_normal((6, int(np.prod(P))))
    np.testing.assert_allclose(oracle.alg1(X, Fs), shuffle_algorithm(X, Fs), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.alg1(X, Fs), X @ np_kron(Fs), rtol=1e-12, atol=1e-12)


def test_alg1_config_A_exact():
    # config A: M=16, two 4x4 factors; fp64 small-integer data -> exact vs brute force.
    seed = synth.SEED_BASE + 0
    X = synth.matrix(16, 16, seed, 0, "int")
    Fs = synth.factors([4, 4], [4, 4], seed, "int")
    assert np.array_equal(oracle.alg1(X, Fs), X @ np_kron(Fs))


def test_identity_factors():
    X = np.random.default_rng(1).standard_normal((4, 2 * 3 * 4))
    Fs = [np.eye(2), np.eye(3), np.eye(4)]
    assert np.array_equal(oracle.alg1(X, Fs), X)


def test_permutation_factors():
    rng = np.random.default_rng(2)
    P = [3, 4, 2]
    perms = [rng.permutation(p) for p in P]
    Fs = [np.eye(p)[perm] for p, perm in zip(P, perms)]  # F[r, c] = 1 iff r == perm^{-1}... rows permuted
    X = rng.standard_normal((3, int(np.prod(P))))
    Y = oracle.alg1(X, Fs)
    K = int(np.prod(P))
    for c in range(K):
        digits = np.unravel_index(c, P)  # F1 most significant
        r_digits = [int(np.nonzero(F[:, d])[0][0]) for F, d in zip(Fs, digits)]  # unique row with a 1
        r = int(np.ravel_multi_index(r_digits, P))
        assert np.array_equal(Y[:, c], X[:, r])


def test_diagonal_factors():
    rng = np.random.default_rng(4)
    P = [2, 4, 3]
    ds = [2.0 ** rng.integers(-3, 4, size=p) for p in P]
    Fs = [np.diag(d) for d in ds]
    X = rng.standard_normal((3, int(np.prod(P))))
    Y = oracle.alg1(X, Fs)
    scale = functools.reduce(np.kron, ds)
    assert np.array_equal(Y, X * scale)


def test_one_hot_rows():
    P, Q = [3, 2, 4], [2, 5, 3]
    Fs = [np.random.default_rng(9 + i).standard_normal((p, q)) for i, (p, q) in enumerate(zip(P, Q))]
    K, L = int(np.prod(P)), int(np.prod(Q))
    rows = [0, 5, K - 1]
    X = np.zeros((len(rows), K))
    for i, r in enumerate(rows):
        X[i, r] = 1.0
    Y = oracle.alg1(X, Fs)
    for i, r in enumerate(rows):
        rd = np.unravel_index(r, P)
        for c in range(L):
            cd = np.unravel_index(c, Q)
            v = Fs[0][rd[0], cd[0]] * Fs[1][rd[1], cd[1]] * Fs[2][rd[2], cd[2]]
            assert Y[i, c] == pytest.approx(v, rel=1e-14, abs=1e-300)


def test_rank1_rows():
    rng = np.random.default_rng(12)
    P, Q = [2, 3, 4], [3, 2, 2]
    Fs = [rng.standard_normal((p, q)) for p, q in zip(P, Q)]
    a = [rng.standard_normal(p) for p in P]
    X = np_kron(a)[None, :]
    expect = np_kron([ai @ Fi for ai, Fi in zip(a, Fs)])
    np.testing.assert_allclose(oracle.alg1(X, Fs)[0], expect, rtol=1e-12, atol=1e-12)


def test_mixed_product_identity():
    # (A(x)B)(C(x)D) = AC (x) BD:  KM(KM(X,{F_i}),{G_i}) == KM(X,{F_i G_i})
    P, R, Q = [2, 3, 2], [3, 2, 2], [2, 2, 3]
    Fs = int_factors(P, R, seed=21)
    Gs = int_factors(R, Q, seed=22)
    X = np.random.default_rng(23).integers(-2, 3, size=(4, int(np.prod(P)))).astype(np.float64)
    lhs = oracle.alg1(oracle.alg1(X, Fs), Gs)
    rhs = oracle.alg1(X, [F @ G for F, G in zip(Fs, Gs)])
    assert np.array_equal(lhs, rhs)


def test_single_factor_is_gemm():
    rng = np.random.default_rng(31)
    F = rng.standard_normal((7, 5))
    X = rng.standard_normal((9, 7))
    np.testing.assert_allclose(oracle.alg1(X, [F]), X @ F, rtol=1e-13, atol=1e-13)
    Fi = rng.integers(-3, 4, size=(7, 5)).astype(np.float64)
    Xi = rng.integers(-3, 4, size=(9, 7)).astype(np.float64)
    assert np.array_equal(oracle.alg1(Xi, [Fi]), Xi @ Fi)


def test_linearity_power_of_two():
    rng = np.random.default_rng(41)
    Fs = [rng.standard_normal((3, 3)), rng.standard_normal((2, 4))]
    X = rng.standard_normal((3, 6))
    assert np.array_equal(oracle.alg1(8.0 * X, Fs), 8.0 * oracle.alg1(X, Fs))


def test_widths_mixed_shapes_reading_G2():
    # P=[8,2], Q=[2,8]: widths K=16 -> 16/2*8=64 -> 64/8*2=16; the max interior width is 64 (G2).
    assert oracle.widths([8, 2], [2, 8]) == [16, 64, 16]
    assert oracle.widths([8] * 6, [8] * 6) == [8 ** 6] * 7
    assert oracle.widths([64, 64, 64], [32, 32, 32]) == [2 ** 15, 2 ** 16, 2 ** 17, 2 ** 18]


def test_row_subset_matches_full_rows():
    seed = synth.SEED_BASE + 99
    M, P = 40, [4, 4, 4]
    X = synth.matrix(M, 64, seed, 0, "urand")
    Fs = synth.factors(P, P, seed, "urand")
    rows = synth.row_subset(M, extra=5)
    Y = oracle.alg1(X, Fs)
    Ys = oracle.alg1(synth.rows_of(rows, 64, seed, 0, "urand"), Fs)
    assert np.array_equal(Ys, Y[rows])


def test_mac_count_closed_form():
    # Algorithm 1 performs M*P*sum_i Q^{N-i} P^i MACs; for P=Q this is N*M*P*K.
    M, P, N = 3, 4, 3
    W = oracle.widths([P] * N, [P] * N)
    macs = sum(M * W[f] * P for f in range(1, N + 1))  # each output of iteration f costs P MACs
    assert macs == N * M * P * P ** N
    assert macs == M * P * sum(P ** (N - i) * P ** i for i in range(1, N + 1))


# ------------------------------------------------------------------ index maps


def test_fused_store_fixtures():
    for K, P, TileK, Fused, bidy, c, expect in golden_rows("fused_store.txt"):
        assert oracle.fused_store_col(int(K), int(P), int(TileK), int(Fused), int(bidy), int(c)) == int(expect)


def test_fused_store_equals_two_unfused_passes():
    # Fig 6: X_{1x256}, 4x4 factors, TileK=128, Fused=2.  Two in-tile sliced multiplies
    # followed by StoreFusedShMem equal the first two iterations of Algorithm 1 on the whole row.
    rng = np.random.default_rng(51)
    X = rng.standard_normal((1, 256))
    F4, F3 = rng.standard_normal((4, 4)), rng.standard_normal((4, 4))
    ref = oracle.sliced_multiply(oracle.sliced_multiply(X, F4), F3)[0]
    out = np.full(256, np.nan)
    for bidy in range(2):
        tile = X[:, bidy * 128:(bidy + 1) * 128]
        t = oracle.sliced_multiply(oracle.sliced_multiply(tile, F4), F3)[0]
        for c in range(128):
            out[oracle.fused_store_col(256, 4, 128, 2, bidy, c)] = t[c]
    np.testing.assert_allclose(out, ref, rtol=1e-14, atol=1e-14)
    # generalized map used by the CUDA path's design (a6): c = u*R + t -> u*(W/C) + g0 + t
    for bidy in range(2):
        for c in range(128):
            u, t = divmod(c, 128 // 16)
            assert oracle.fused_store_col(256, 4, 128, 2, bidy, c) == u * (256 // 16) + bidy * 8 + t


def test_shift_caching_fixtures():
    for k, TileP, RegK, expect in golden_rows("shift_caching.txt"):
        assert oracle.shift_pos(int(k), int(TileP), int(RegK)) == int(expect)
    # the map is a permutation within each slice (a load/store round trip is lossless)
    for TileP, RegK in [(4, 2), (8, 1), (8, 4), (16, 2)]:
        pos = [oracle.shift_pos(k, TileP, RegK) for k in range(TileP * 32)]
        assert sorted(pos) == list(range(TileP * 32))


# ------------------------------------------------------------------ O3: Algorithm 2


def test_grid_rule():
    for G, GM, GK in golden_rows("grid_rule.txt"):
        got = oracle.grid(int(G))
        if int(GM) == 0:
            assert got is None
        else:
            assert got == (int(GM), int(GK))


def test_alg2_ledger_fixtures():
    for M, N, P, GM, GK, local, total in golden_rows("comm_ledger.txt"):
        M, N, P, GM, GK = int(M), int(N), int(P), int(GM), int(GK)
        local = [int(v) for v in local.split(",")]
        seed = synth.SEED_BASE + 77
        X = synth.matrix(M, P ** N, seed, 0, "urand")
        Fs = synth.factors([P] * N, [P] * N, seed, "urand")
        Y, ledger = oracle.alg2(X, Fs, GM, GK, local)
        assert sum(ledger) == int(total)
        np.testing.assert_allclose(Y, oracle.alg1(X, Fs), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("GM,GK,P,Q,local", [
    (1, 4, [4] * 4, [4] * 4, [2, 2]),
    (2, 2, [4] * 4, [4] * 4, [3, 1]),
    (4, 1, [4] * 3, [4] * 3, [3]),
    (1, 2, [16] * 3, [16] * 3, [2, 1]),
    (2, 2, [8, 4, 4], [4, 8, 4], [1, 2]),
    (2, 4, [4] * 5, [4] * 5, [2, 2, 1]),
    (1, 2, [2, 2, 2, 2], [2, 2, 2, 2], [2, 2]),
])
def test_alg2_gather_equals_alg1(GM, GK, P, Q, local):
    seed = synth.SEED_BASE + 5
    M = 4 * GM
    X = synth.matrix(M, int(np.prod(P)), seed, 0, "int")
    Fs = synth.factors(P, Q, seed, "int")
    Y, ledger = oracle.alg2(X, Fs, GM, GK, local)
    assert np.array_equal(Y, oracle.alg1(X, Fs))
    # ledger = sum over rounds of M * W_j * (1 - 1/GK)  (reading G12)
    W = oracle.widths(P, Q)
    f, expect = len(P), []
    for n in local:
        f -= n
        expect.append(M * W[f] * (GK - 1) // GK)
    assert ledger == expect


def test_alg2_rejects_illegal_round():
    # {1,4}, K=256, P=4: Local_max = floor(log_4 64) = 3; four local multiplies in one round is illegal.
    seed = synth.SEED_BASE + 6
    X = synth.matrix(1, 256, seed, 0, "urand")
    Fs = synth.factors([4] * 4, [4] * 4, seed, "urand")
    with pytest.raises(ValueError):
        oracle.alg2(X, Fs, 1, 4, [4])


def test_fig8_local_layout():
    # Fig 8: {1,4}, X_{1x256}, four 4x4, Local=2: after two local multiplies each GPU's local
    # intermediate holds 16 elements for every GPU, as runs of 4 contiguous global columns.
    rng = np.random.default_rng(61)
    X = rng.standard_normal((1, 256))
    F4, F3 = rng.standard_normal((4, 4)), rng.standard_normal((4, 4))
    glob = oracle.sliced_multiply(oracle.sliced_multiply(X, F4), F3)[0]
    where = {v: i for i, v in enumerate(glob)}
    assert len(where) == 256  # values distinct
    for gK in range(4):
        loc = oracle.sliced_multiply(oracle.sliced_multiply(X[:, gK * 64:(gK + 1) * 64], F4), F3)[0]
        # same arithmetic on the same slices -> bit-identical values
        cols = [where[v] for v in loc]
        for d in range(4):
            part = cols[16 * d:16 * (d + 1)]
            assert all(64 * d <= c < 64 * (d + 1) for c in part)  # destined to GPU d
            for r in range(4):
                run = part[4 * r:4 * r + 4]
                assert run == list(range(run[0], run[0] + 4))  # runs of 4 contiguous columns
