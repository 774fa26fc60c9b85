#!/usr/bin/env python
"""Experiment: config E's K-split rounds on the virtual backend (all ranks of a {GM,GK} grid in this process on one
GPU, device-copy exchange), ms per call; run once with and once without KRON_NO_HANDOFF=1 to compare the v11
tile-major rounds with the direct-index ones.

    python tools/exp_dist_virtual.py [M] [GK]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2401_10187_b200 import kron  # noqa: E402


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    GK = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    dev = torch.device("cuda:0")
    P = [16] * 5
    K = 16 ** 5
    Kl = K // GK
    blocks = []
    for g in range(GK):
        x = torch.empty((M, Kl), dtype=torch.float32, device=dev)
        synth.fill_device(x.data_ptr(), M, Kl, synth.SEED_BASE + 5 + g, 0, "urand", np.float32)
        blocks.append(x)
    Fs = [torch.from_numpy(f).to(dev) for f in synth.factors(P, P, synth.SEED_BASE + 5, "urand", np.float32)]
    ctx = kron.DistContext("virtual", GM=1, GK=GK, chunks=2)
    outs = [torch.empty((M, Kl), dtype=torch.float32, device=dev) for _ in range(GK)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        kron.matmul_dist(M, blocks, Fs, ctx, out=outs)
    torch.cuda.synchronize()
    n = 5
    e0.record()
    for _ in range(n):
        kron.matmul_dist(M, blocks, Fs, ctx, out=outs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"M={M} GK={GK} handoff={'off' if os.environ.get('KRON_NO_HANDOFF') else 'on'}: {ms:.3f} ms per call "
          f"({ms / GK:.3f} ms per rank), checksum {float(outs[0][::37, ::4099].double().sum()):.6e}", flush=True)
    if os.environ.get("PROF"):
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            kron.matmul_dist(M, blocks, Fs, ctx, out=outs)
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
    ctx.close()


if __name__ == "__main__":
    main()
