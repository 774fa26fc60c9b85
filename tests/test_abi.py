"""CPU tests of the C-ABI library: it loads, exports every symbol include/kron.h declares, rejects bad
arguments synchronously, and its host-side planner (pass plan, costs, distributed round plan) obeys
the paper's rules.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kron():
    from paper_2401_10187_b200 import build
    build.build()
    from paper_2401_10187_b200 import kron as k
    return k


def header_symbols():
    with open(os.path.join(ROOT, "include", "kron.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kron_[a-z_0-9]+)\s*\(", text)))


def test_exports_every_declared_symbol(kron):
    syms = header_symbols()
    assert "kron_matmul" in syms and "kron_matmul_dist" in syms and len(syms) >= 12
    lib = ctypes.CDLL(kron.lib_path)
    for s in syms:
        assert hasattr(lib, s), f"libkron.so does not export {s}"


def test_status_strings(kron):
    lib = kron.raw_lib()
    for code, name in kron.STATUS.items():
        assert lib.kron_status_string(code).decode() == name


def _call(kron, M, P, Q, dtype=0, X=1, F=True, Y=1):
    lib = kron.raw_lib()
    n = len(P)
    Pa = (ctypes.c_int32 * max(n, 1))(*P) if n else None
    Qa = (ctypes.c_int32 * max(n, 1))(*Q) if n else None
    Fp = (ctypes.c_void_p * max(n, 1))(*([1] * n)) if F else None
    return lib.kron_matmul(M, n, Pa, Qa, X, Fp, Y, dtype, None)


def test_argument_errors_are_synchronous(kron):
    assert _call(kron, 4, [2, 2], [2, 2], X=None) == 1      # null X
    assert _call(kron, 4, [2, 2], [2, 2], F=False) == 1     # null F
    assert _call(kron, 4, [], []) == 1                      # N < 1
    assert _call(kron, 4, [2, 0], [2, 2]) == 1              # P_i < 1
    assert _call(kron, 4, [2, 2], [2, -1]) == 1             # Q_i < 1
    assert _call(kron, 4, [2, 2], [2, 2], dtype=7) == 1     # bad dtype
    assert _call(kron, -1, [2, 2], [2, 2]) == 1             # M < 0
    assert _call(kron, 4, [2 ** 30] * 3, [2] * 3) == 2      # prod P overflows
    assert _call(kron, 0, [2, 2], [2, 2], X=None, Y=None) == 0  # M = 0: no-op


def test_plan_configs(kron):
    f32, f64 = "float32", "float64"
    # config B: 6 x (8x8) fp32 -> two fused passes of 3 (Fused = 3 at B200 capacity)
    assert kron.plan_describe(1024, [8] * 6, [8] * 6, f32) == [(6, 3, "fused"), (3, 3, "fused")]
    # config C: 4 x (32x32) -> (2,2) in fp32 and fp64
    assert kron.plan_describe(1024, [32] * 4, [32] * 4, f32) == [(4, 2, "fused"), (2, 2, "fused")]
    assert kron.plan_describe(1024, [32] * 4, [32] * 4, f64) == [(4, 2, "fused"), (2, 2, "fused")]
    # config A: K = 16 is narrower than one 128-byte TMA line -> generic
    # config A: rows of 16 are too short for the TMA kernels; both factors fuse in one chain pass (chain.cu)
    assert kron.plan_describe(16, [4, 4], [4, 4], f32) == [(2, 2, "chain")]
    # every plan applies every factor exactly once, N -> 1
    for P, Q, dt in [([16] * 5, [16] * 5, f32), ([128] * 3, [128] * 3, f64), ([64] * 3, [32] * 3, f64),
                     ([3, 8, 8, 8, 5], [4, 8, 8, 8, 2], f32), ([2] * 12, [2] * 12, f64)]:
        plan = kron.plan_describe(64, P, Q, dt)
        covered = []
        for first, nf, _ in plan:
            covered += list(range(first, first - nf, -1))
        assert covered == list(range(len(P), 0, -1))


def test_plan_cost_closed_forms(kron):
    # FLOPs = sum_f 2 M W_f Q_f (north_star); for square factors = 2 N M P K
    b, fl = kron.plan_cost(1024, [8] * 6, [8] * 6, "float32")
    assert fl == 2 * 6 * 1024 * 8 * 8 ** 6
    # bytes of the (3,3) plan: two passes, each reads and writes M*K fp32, plus the factors
    assert b == 2 * 2 * 4 * 1024 * 8 ** 6 + 6 * 4 * 64
    W = oracle.widths([64] * 3, [32] * 3)
    _, fl2 = kron.plan_cost(320, [64] * 3, [32] * 3, "float64")
    assert fl2 == sum(2 * 320 * W[f] * 32 for f in range(1, 4))


def test_workspace_sizes(kron):
    # one pass: no workspace; P = Q: Y doubles as the other ping-pong buffer -> one M x K buffer
    assert kron.workspace_size(16, [4], [4], "float32") == 0
    assert kron.workspace_size(1024, [8] * 6, [8] * 6, "float32") == 1024 * 8 ** 6 * 4
    # mixed widths (G2): interior width 64 > L = 16 needs the workspace sized by the widest interior
    ws = kron.workspace_size(10, [8, 2], [2, 8], "float64")
    assert ws >= 10 * 64 * 8


def test_grid_rule_matches_oracle(kron):
    for G in [1, 2, 4, 8, 16, 32, 64]:
        assert kron.grid_rule(G) == oracle.grid(G)
    with pytest.raises(kron.KronError):
        kron.grid_rule(6)


@pytest.mark.parametrize("M,P,Q,GM,GK", [
    (1, [4] * 4, [4] * 4, 1, 4),
    (8, [16] * 5, [16] * 5, 4, 2),
    (4, [16] * 5, [16] * 5, 2, 2),
    (4, [4] * 5, [4] * 5, 2, 4),
    (6, [8, 4, 4], [4, 8, 4], 2, 2),
    (2, [2] * 6, [2] * 6, 1, 4),
])
def test_dist_plan_legal_and_ledger_matches_oracle(kron, M, P, Q, GM, GK):
    rounds, ledger = kron.dist_plan(M, P, Q, GM, GK)
    assert sum(rounds) == len(P)
    seed = synth.SEED_BASE + 11
    X = synth.matrix(M, int(np.prod(P)), seed, 0, "int")
    Fs = synth.factors(P, Q, seed, "int")
    Y, oled = oracle.alg2(X, Fs, GM, GK, rounds)  # the oracle simulator rejects illegal rounds
    assert oled == ledger
    assert np.array_equal(Y, oracle.alg1(X, Fs))


def test_dist_plan_paper_local(kron):
    # Fig 8 / Alg 2: {1,4}, K = 256, P = 4 -> Local_max = floor(log_4 64) = 3; N = 4 -> 2 rounds,
    # ledger 2 * 256 * 3/4 = 384
    rounds, ledger = kron.dist_plan(1, [4] * 4, [4] * 4, 1, 4)
    assert len(rounds) == 2 and sum(ledger) == 384
    # config E at the paper grid {4,2}: Local_max = floor(log_16 2^19) = 4, N = 5 -> 2 exchanges
    rounds, ledger = kron.dist_plan(4096, [16] * 5, [16] * 5, 4, 2)
    assert len(rounds) == 2 and sorted(rounds) == [2, 3]
    with pytest.raises(kron.KronError):
        kron.dist_plan(4095, [16] * 5, [16] * 5, 4, 2)  # GM does not divide M


def test_autotune_candidates(kron):
    # the autotuner times alternative plans; the static plan is always one of them
    assert kron.autotune_candidates(1024, [8] * 6, [8] * 6, "float32") >= 3   # fusion caps 3/2/1 + families
    assert kron.autotune_candidates(1024, [32] * 4, [32] * 4, "float64") >= 2  # + DMMA on/off
    assert kron.autotune_candidates(16, [4, 4], [4, 4], "float32") == 2       # one chain pass or two generic
    assert kron.autotune_candidates(0, [8] * 2, [8] * 2, "float32") == 0
    lib = kron.raw_lib()
    Pa = (ctypes.c_int32 * 2)(2, 2)
    assert lib.kron_autotune(4, 2, Pa, Pa, None, None, None, 0, 3, None, None, None) == 1  # null buffers
    assert lib.kron_plan_cache_clear() == 0


def test_plan_kernels(kron):
    # the kernel family of every pass (bench.py's roofline label, ncu_traffic keys)
    assert kron.plan_kernels(1024, [8] * 6, [8] * 6, "float32") == ["kron_fused_pipe_kernel"] * 2
    assert kron.plan_kernels(1024, [32] * 4, [32] * 4, "float64") == ["kron_fused_dmma2_kernel"] * 2
    assert kron.plan_kernels(320, [128] * 3, [128] * 3, "float64") == ["kron_dmma_kernel"] * 3
    assert kron.plan_kernels(16, [4, 4], [4, 4], "float32") == ["kron_chain_kernel"]
    lib = kron.raw_lib()
    Pa = (ctypes.c_int32 * 2)(4, 4)
    buf = ctypes.create_string_buffer(8)
    assert lib.kron_plan_kernel(16, 2, Pa, Pa, 0, 5, buf, 8) == 1   # no such pass


def test_handoff_plans(kron):
    # v11: a [16^3 triple, 16^2 pair] plan passes its intermediate tile-major (fused.cu kron_tri_tm_kernel); other
    # plans, the tensor-core modes and three-factor plans keep the direct-index layout
    assert kron.plan_kernels(4096, [16] * 5, [16] * 5, "float32") == ["kron_tri_tm_kernel", "kron_pair_tm_kernel"]
    assert kron.plan_kernels(5, [16] * 5, [16] * 5, "float32") == ["kron_tri_tm_kernel", "kron_pair_tm_kernel"]
    assert kron.plan_kernels(64, [16] * 6, [16] * 6, "float32") == ["kron_fused_gemm3c_kernel"] * 2
    assert "kron_tri_tm_kernel" not in kron.plan_kernels(64, [16] * 3, [16] * 3, "float32")
    assert kron.plan_kernels(64, [8, 16, 16, 16, 16, 16], [8, 16, 16, 16, 16, 16], "float32")[0] != "kron_tri_tm_kernel"
    # same workspace as the direct-index plan; the autotuner also times the plan without the hand-off
    assert kron.workspace_size(64, [16] * 5, [16] * 5, "float32") == 64 * 16 ** 5 * 4
    assert kron.autotune_candidates(64, [16] * 5, [16] * 5, "float32") >= 2


def test_tensor_core_mode_plans(kron):
    # the tensor-core modes (dtype codes 2 = 3xTF32, 3 = TF32) route the P = 16 / 32 fp32 square pairs to the
    # tcgen05 kernel (tc.cu); other passes stay on the fp32 CUDA-core kernels; fp64 data rejects the modes
    for mode in ("3xtf32", "tf32"):
        assert kron.plan_kernels(1024, [32] * 4, [32] * 4, "float32", mode) == ["kron_tc_pair_kernel"] * 2
        assert kron.plan_kernels(1024, [8] * 6, [8] * 6, "float32", mode) == ["kron_fused_pipe_kernel"] * 2
        # config E: the 16x16 triple stays on the CUDA cores, the pair goes to the tensor cores
        assert kron.plan_kernels(64, [16] * 5, [16] * 5, "float32", mode) == ["kron_fused_gemm3c_kernel",
                                                                              "kron_tc_pair_kernel"]
        assert kron.workspace_size(1024, [32] * 4, [32] * 4, "float32", mode) == \
            kron.workspace_size(1024, [32] * 4, [32] * 4, "float32")
        with pytest.raises(ValueError):
            kron.dtype_code("float64", mode)
    assert kron.dtype_code("float32", "tf32") == 3 and kron.dtype_code("float32", "3xtf32") == 2
    assert _call(kron, 4, [2, 2], [2, 2], dtype=4) == 1   # unknown dtype code


def test_graph_argument_errors(kron):
    # kron_graph_create validates synchronously (nothing is captured on bad arguments)
    lib = kron.raw_lib()
    Pa = (ctypes.c_int32 * 2)(4, 4)
    h = ctypes.c_void_p()
    assert lib.kron_graph_create(4, 2, Pa, Pa, None, None, None, 0, None, 0, ctypes.byref(h)) == 1
    assert lib.kron_graph_create(0, 2, Pa, Pa, 1, None, 1, 0, None, 0, ctypes.byref(h)) == 1  # M = 0
    assert lib.kron_graph_launch(None, None) == 1
    assert lib.kron_graph_destroy(None) == 0


def test_table4_shapes_plan_and_autotune(kron):
    # every paper Table 4 shape (odd M, odd / mixed / non-square factors) gets a legal plan, and the
    # autotuner has at least one candidate for it (Table 4)
    import bench
    for M, P, Q in bench.TABLE4:
        for dt in ("float32", "float64"):
            plan = kron.plan_describe(M, P, Q, dt)
            covered = []
            for first, nf, _ in plan:
                covered += list(range(first, first - nf, -1))
            assert covered == list(range(len(P), 0, -1))
            assert kron.autotune_candidates(M, P, Q, dt) >= 1
            assert len(kron.plan_kernels(M, P, Q, dt)) == len(plan)


def test_host_path_argument_errors(kron):
    lib = kron.raw_lib()
    Pa = (ctypes.c_int32 * 2)(4, 4)
    assert lib.kron_matmul_host(4, 2, Pa, Pa, None, None, None, 0, 0, None) == 1     # null buffers
    Fp = (ctypes.c_void_p * 2)(1, 1)
    assert lib.kron_matmul_host(4, 2, Pa, Pa, 1, Fp, 1, 0, -1, None) == 1           # chunk_rows < 0
    assert lib.kron_matmul_host(0, 2, Pa, Pa, None, None, None, 0, 0, None) == 0     # M = 0: no-op


def test_dist_round_info_fused_layouts(kron):
    # host-only: which rounds of backends 0 / 1 write the send buffer from the last pass's epilogue (fused
    # pack) and read the previous receive buffer through the StoreGPUTile-ordered tensor map (fused remap)
    ctx = kron.DistContext("virtual", GM=4, GK=2)
    # config E on the 8-GPU paper grid: round 1 = v9 triple (no remap: it reads X), round 2 = v6 pair
    assert ctx.round_info(4096, [16] * 5, [16] * 5, "float32") == [(True, False), (True, True)]
    # C32 on {1,2}: two rounds of v6 P = 32 pairs
    ctx2 = kron.DistContext("virtual", GM=1, GK=2)
    assert ctx2.round_info(1024, [32] * 4, [32] * 4, "float32") == [(True, False), (True, True)]
    # fp64 pairs (DMMA v5) have no pushing epilogue -> pack kernel, but read the receive buffer in place
    assert ctx2.round_info(1024, [32] * 4, [32] * 4, "float64") == [(False, False), (False, True)]
    # the fused layouts can be switched off (separate pack / StoreGPUTile kernels)
    ctx3 = kron.DistContext("virtual", GM=1, GK=2, fused=False)
    assert ctx3.round_info(1024, [32] * 4, [32] * 4, "float32") == [(False, False), (False, False)]
    with pytest.raises(kron.KronError):
        kron.DistContext("virtual", GM=1, GK=2, chunks=0)
    # exchange layouts: config E's rounds on the v11 tile-major layouts (fp32 only, fused layouts on), the rest
    # direct-index or plain
    assert ctx.round_layouts(4096, [16] * 5, [16] * 5, "float32") == ["tile-major", "tile-major"]
    assert ctx.round_layouts(4096, [16] * 5, [16] * 5, "float64") != ["tile-major", "tile-major"]
    assert ctx2.round_layouts(1024, [32] * 4, [32] * 4, "float32") == ["direct-index", "direct-index"]
    assert ctx3.round_layouts(4096, [16] * 5, [16] * 5, "float32") == ["plain", "plain"]
    ctx8 = kron.DistContext("virtual", GM=1, GK=8)
    assert ctx8.round_layouts(64, [16] * 5, [16] * 5, "float32") == ["tile-major", "tile-major"]
    for c in (ctx, ctx2, ctx3, ctx8):
        c.close()


def test_chain_plans_for_odd_p(kron):
    # square factors of any size P fuse through chain.cu (Fused <= floor(log_P TileK)): the paper's Table 4
    # shapes 3^7 (one pass of 7) and 6^7 (4 + 3); power-of-2 P keeps the TMA kernels
    assert kron.plan_describe(1024, [3] * 7, [3] * 7, "float32") == [(7, 7, "chain")]
    assert kron.plan_describe(1024, [6] * 7, [6] * 7, "float32") == [(7, 4, "chain"), (3, 3, "chain")]
    assert kron.plan_kernels(1024, [4] * 7, [4] * 7, "float32") == ["kron_fused_warp_kernel", "kron_fused_pipe_kernel"]
    # the autotuner searches the chain tile size (R / 1, 2, 4 chunks per tile) besides the plan families
    assert kron.autotune_candidates(1024, [6] * 7, [6] * 7, "float32") >= 3
