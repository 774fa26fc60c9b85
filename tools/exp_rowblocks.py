#!/usr/bin/env python
"""Experiment: config E in row blocks (both passes per block, so the pair reads the block's intermediate while it
is still in L2) vs the whole matrix per pass.  Prints ms per step per block size.

    python tools/exp_rowblocks.py [block sizes...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2401_10187_b200 import kron  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    M, P = 4096, [16] * 5
    K = 16 ** 5
    X = torch.empty((M, K), dtype=torch.float32, device=dev)
    synth.fill_device(X.data_ptr(), M, K, synth.SEED_BASE + 5, 0, "urand", np.float32)
    Fs = [torch.from_numpy(f).to(dev) for f in synth.factors(P, P, synth.SEED_BASE + 5, "urand", np.float32)]
    Y = torch.empty_like(X)
    blocks = [int(b) for b in sys.argv[1:]] or [4096, 64, 32, 16, 8]
    ws = torch.empty(kron.workspace_size(M, P, P, torch.float32), dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ref = None
    for b in blocks:
        def step():
            for r0 in range(0, M, b):
                kron.matmul_ws(X[r0:r0 + b], Fs, Y[r0:r0 + b], ws)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0.record()
        n = 5
        for _ in range(n):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        s = float(Y[::97, ::4099].double().sum())
        ref = s if ref is None else ref
        print(f"block {b:5d}: {ms:8.3f} ms per step  (checksum {'ok' if s == ref else 'DIFF'})", flush=True)


if __name__ == "__main__":
    main()
