"""World-size-2 CPU (gloo) test of the distributed host logic (-m "not gpu").

Two real processes play the ranks of a {1,2} and a {2,1} grid.  Each asks libkron's host planner for
the round plan (kron_dist_plan: must agree across ranks), performs each round's local sliced
multiplies on its block with the ORACLE (test-only arithmetic), packs the destination-major send
buffer, exchanges it with torch.distributed.all_to_all_single over gloo, and applies the StoreGPUTile
placement documented in include/kron.h / dist.cu.  The gathered result must equal Algorithm 1, and
the values each rank sent must match the ledger (reading G12).  This pins the protocol that
the CUDA pack / StoreGPUTile kernels and the NCCL all-to-all implement.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, GM, GK, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2401_10187_b200 import kron
        M, P = 4, [4] * 4
        K = 4 ** 4
        seed = synth.SEED_BASE + 400
        X = synth.matrix(M, K, seed, 0, "int")
        Fs = synth.factors(P, P, seed, "int")
        rounds, ledger = kron.dist_plan(M, P, P, GM, GK)
        allr = [None] * world
        dist.all_gather_object(allr, (rounds, ledger))
        assert all(a == (rounds, ledger) for a in allr)
        gm, gk = rank // GK, rank % GK
        Ml, W = M // GM, K
        T = X[gm * Ml:(gm + 1) * Ml, gk * (W // GK):(gk + 1) * (W // GK)]
        f, sent = len(P), 0
        for k in rounds:
            C = int(np.prod(P[f - k:f]))
            Qc = int(np.prod(P[f - k:f]))
            wl = T.shape[1]
            for i in range(k):  # local sliced multiplies (oracle arithmetic)
                T = oracle.sliced_multiply(T, Fs[f - 1 - i])
            rho = wl // C
            B = T.shape[1] // GK
            send = np.concatenate([T[:, d * B:(d + 1) * B].reshape(-1) for d in range(GK)])
            recv = np.empty_like(send)
            sent += send.size - B * Ml
            # row group = ranks with the same gm; gloo all_to_all over the whole world only when GM == 1
            if GK > 1:
                st, rt = torch.from_numpy(send), torch.from_numpy(recv)
                dist.all_to_all_single(rt, st)
                recv = rt.numpy()
            else:
                recv = send
            nxt = np.empty_like(T)
            wl2 = T.shape[1]
            for src in range(GK):
                part = recv[src * Ml * B:(src + 1) * Ml * B].reshape(Ml, B)
                for e in range(Qc // GK):
                    for t in range(rho):
                        nxt[:, (e * GK + src) * rho + t] = part[:, e * rho + t]
            T, f = nxt, f - k
            assert wl2 == nxt.shape[1]
        ref = oracle.alg1(X, Fs)
        L = ref.shape[1]
        ok = np.array_equal(T, ref[gm * Ml:(gm + 1) * Ml, gk * (L // GK):(gk + 1) * (L // GK)])
        tot = [0] * world
        dist.all_gather_object(tot, sent)
        q.put((rank, ok, sum(tot), sum(ledger)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("GM,GK", [(1, 2), (2, 1)])
def test_gloo_world2_protocol(GM, GK):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, GM, GK, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted(q.get(timeout=5) for _ in range(2))
    for rank, ok, sent, ledger in res:
        assert ok, f"rank {rank}: distributed result differs from Algorithm 1"
        assert sent == ledger
    assert all(p.exitcode == 0 for p in procs)
