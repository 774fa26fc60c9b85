#!/usr/bin/env python
"""Small-shape runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2401_10187_b200 import kron  # noqa: E402

CASES = [
    (9, [8] * 6, [8] * 6, np.float32),          # v3 factor pipeline (3,3)
    (2, [32] * 3, [32] * 3, np.float32),        # P = 32 chunk pair (v12 since round 2) (+ v2)
    (3, [8, 16, 16, 16], [8, 16, 16, 16], np.float32),  # v9 16x16 triple on a CTA pair (DSMEM) + v2
    (2, [16] * 4, [16] * 4, np.float32),        # v6, P = 16 (64-chunk tiles)
    (2, [16] * 3, [16] * 3, np.float32),        # v4/v6 (2) + v2 (1)
    (2, [32] * 3, [32] * 3, np.float64),        # v5 DMMA chunk pair (+ v2)
    (3, [16] * 2, [16] * 2, np.float64),        # v4 fp64
    (2, [64] * 3, [32] * 3, np.float64),        # v7 64x32 pair on DMMA + DMMA gemm
    (5, [4] * 5, [4] * 5, np.float64),          # v3 fp64 / v2
    (3, [16] * 3, [16] * 3, np.float64),        # v1/v2 fp64
    (2, [64, 64], [64, 64], np.float64),        # DMMA gemm (32-column tiles)
    (2, [128, 128], [128, 128], np.float64),    # DMMA gemm (128-column tiles)
    (2, [64, 64], [64, 64], np.float32),        # FFMA2 gemm
    (3, [3, 5], [4, 2], np.float32),            # generic
    # round 2
    (3, [8, 16, 16, 16], [8, 16, 16, 16], np.float32, None),    # v10 triple (constant-bank FFMA2, groups of 4)
    (2, [16] * 4, [16] * 4, np.float32, None),                  # v10 pair
    (3, [3] * 5, [3] * 5, np.float32, None),                    # chain (odd P, one pass)
    (2, [6] * 5, [6] * 5, np.float64, None),                    # chain (even chunk, padded, cp.async 16 B)
    (17, [32] * 3, [32] * 3, np.float32, "tf32"),               # tcgen05 pair, TF32
    (17, [32] * 3, [32] * 3, np.float32, "3xtf32"),             # tcgen05 pair, 3xTF32
    (5, [32, 16, 16], [32, 16, 16], np.float32, "3xtf32"),      # tcgen05 pair, P = 16
    # round 2, second half
    (3, [16] * 5, [16] * 5, np.float32, None),                  # v11 triple -> pair (tile-major hand-off)
    (2, [32] * 4, [32] * 4, np.float32, None),                  # v12 P = 32 pairs (F1 in the constant bank)
    (9, [32] * 4, [32] * 4, np.float32, "3xtf32"),              # tcgen05 pair v2 (two groups, polled MMAs)
]


def main():
    dev = torch.device("cuda:0")
    for case in CASES:
        M, P, Q, dt = case[:4]
        mode = case[4] if len(case) > 4 else None
        seed = synth.SEED_BASE + 77
        X = synth.matrix(M, int(np.prod(P)), seed, 0, "urand", dt)
        Fs = synth.factors(P, Q, seed, "urand", dt)
        Y = kron.matmul(torch.from_numpy(X).to(dev), [torch.from_numpy(f).to(dev) for f in Fs], mode=mode)
        torch.cuda.synchronize()
        print("ok", M, P, Q, np.dtype(dt).name, mode, kron.plan_kernels(M, P, Q, np.dtype(dt).name, mode), float(Y.sum()))
    # the autotuner runs every candidate plan of one shape
    X = torch.from_numpy(synth.matrix(2, 16 ** 4, 5, 0, "urand", np.float32)).to(dev)
    _, n, _ = kron.autotune(X, [torch.from_numpy(f).to(dev) for f in synth.factors([16] * 4, [16] * 4, 5, "urand", np.float32)], reps=1)
    torch.cuda.synchronize()
    print("ok autotune", n, "candidates")
    ctx = kron.DistContext("virtual", GM=2, GK=2)
    X = synth.matrix(4, 16 ** 3, 1, 0, "urand", np.float32)
    blocks = [torch.from_numpy(np.ascontiguousarray(X[(r // 2) * 2:(r // 2) * 2 + 2, (r % 2) * 2048:(r % 2) * 2048 + 2048])).to(dev)
              for r in range(4)]
    Fs = [torch.from_numpy(f).to(dev) for f in synth.factors([16] * 3, [16] * 3, 1, "urand", np.float32)]
    kron.matmul_dist(4, blocks, Fs, ctx)
    torch.cuda.synchronize()
    print("ok dist virtual 2x2 (fused send / receive layouts, 2 row chunks)", ctx.round_info(4, [16] * 3, [16] * 3, "float32"))


if __name__ == "__main__":
    main()
