"""Pins for the shared input generator (synth/): published splitmix64 outputs, value ranges,
exact representability in fp32, and host/device twin agreement (device part is -m gpu)."""
import os

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_outputs():
    gamma = 0x9E3779B97F4A7C15
    with open(os.path.join(GOLDEN, "splitmix64.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            i, v = line.split()
            assert synth.splitmix64((int(i) * gamma) % 2 ** 64) == int(v, 16)


def test_modes_ranges_and_fp32_exact():
    seed = synth.SEED_BASE
    u = synth.fill(10000, seed, 0, "urand")
    assert u.min() >= 0 and u.max() < 1
    assert np.array_equal(u.astype(np.float32).astype(np.float64), u)
    s = synth.fill(10000, seed, 0, "srand")
    assert s.min() >= -1 and s.max() < 1 and np.array_equal(s, 2 * u - 1)
    assert set(np.unique(synth.fill(10000, seed, 1, "int"))) == {-2.0, -1.0, 0.0, 1.0, 2.0}
    assert set(np.unique(synth.fill(10000, seed, 1, "int1"))) == {-1.0, 0.0, 1.0}
    assert np.array_equal(synth.fill(100, seed, 0, "urand", np.float32), u[:100].astype(np.float32))


def test_counter_based_offsets_and_rows():
    seed = synth.SEED_BASE + 3
    full = synth.fill(1000, seed, 2, "srand")
    assert np.array_equal(synth.fill(100, seed, 2, "srand", first=500), full[500:600])
    X = synth.matrix(10, 100, seed, 2, "srand")
    assert np.array_equal(synth.rows_of([3, 7], 100, seed, 2, "srand"), X[[3, 7]])
    assert not np.array_equal(synth.fill(100, seed, 3, "srand"), full[:100])  # tensor ids differ


def test_gp_factor_structure():
    F = synth.gp_factor(16, 16)
    assert np.allclose(F, F.T) and np.all(np.diag(F) == 1.0)
    assert np.all(np.linalg.eigvalsh(F) > -1e-12)  # RBF Gram matrix: PSD
    G = synth.gp_factor(64, 32)
    assert G.shape == (64, 32) and G.max() <= 1.0 and G.min() > 0


@pytest.mark.gpu
def test_device_twin_matches_host(cuda_device):
    import torch
    seed = synth.SEED_BASE + 1
    for dt, tdt in ((np.float32, torch.float32), (np.float64, torch.float64)):
        for mode in ("urand", "srand", "int", "int1"):
            x = torch.empty((37, 129), dtype=tdt, device=cuda_device)
            synth.fill_device(x.data_ptr(), 37, 129, seed, 0, mode, dt, r0=5, c0=11, ld=400)
            torch.cuda.synchronize()
            ref = synth.matrix(60, 400, seed, 0, mode, dt)[5:42, 11:140]
            assert np.array_equal(x.cpu().numpy(), ref)
