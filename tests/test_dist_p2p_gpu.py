"""GPU parity of the P2P distributed backend (NEXT-1: Algorithm 2's exchange as one kernel over peer
memory) through kron_matmul_dist.

Real processes play the ranks (one process per rank, gloo process group for the IPC-handle exchange
only).  Only one B200 is available per run, so every rank runs on cuda:0: CUDA IPC maps the other
processes' heaps exactly as it maps a peer GPU's over NVLink, and the device-side flag barriers work
across contexts sharing the GPU.  Each rank's Y_local is compared with the oracle's rows/columns block:
bit-exact on integer data, tolerance on random data.  Two consecutive calls on one context check that
heap halves and barrier epochs carry over between calls.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, GM, GK, M, P, Q, q, push=True):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2401_10187_b200 import kron
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        ctx = kron.DistContext("p2p", GM=GM, GK=GK, push=push)  # push=False: every round via the pull kernel
        gm, gk = ctx.coords()
        K, L = int(np.prod(P)), int(np.prod(Q))
        Ml, Kl, Ll = M // GM, K // GK, L // GK
        res = []
        for dt, mode, call in ((np.float64, "int", 0), (np.float32, "urand", 1), (np.float64, "int", 2)):
            seed = synth.SEED_BASE + 500 + call
            X = synth.matrix(M, K, seed, 0, mode, dt)
            Fs = synth.factors(P, Q, seed, mode, dt)
            xb = torch.from_numpy(np.ascontiguousarray(X[gm * Ml:(gm + 1) * Ml, gk * Kl:(gk + 1) * Kl])).to(dev)
            Y = kron.matmul_dist(M, xb, [torch.from_numpy(f).to(dev) for f in Fs], ctx, check=True)
            torch.cuda.synchronize()
            ref = oracle.alg1(X, Fs)[gm * Ml:(gm + 1) * Ml, gk * Ll:(gk + 1) * Ll]
            y = Y.cpu().numpy()
            if mode == "int":
                res.append(bool(np.array_equal(y, ref.astype(dt))))
            else:
                res.append(float(np.max(np.abs(y - ref) / np.abs(ref))) <= 1e-5)
        timeouts = ctx.timeouts()
        dist.barrier()
        ctx.close()
        q.put((rank, res, timeouts))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, [repr(e)], -1))
    finally:
        dist.destroy_process_group()


GRIDS = [
    # (GM, GK, M, P, Q)
    (1, 2, 4, [16] * 5, [16] * 5),    # config E shapes, K split only (2 rounds; round 1 pushes from v9)
    (2, 2, 4, [16] * 5, [16] * 5),    # paper rule for 4 GPUs on E shapes (push + pull)
    (1, 2, 2, [16] * 4, [16] * 4),    # round 1 = P=16 chunk pairs (v6, 256-byte-run store path) pushing
    (1, 2, 2, [32] * 4, [32] * 4),    # round 1 = P=32 chunk pairs (v6, chunk-octet store path) pushing
    (2, 2, 4, [8] * 4, [8] * 4),      # paper rule for 4 GPUs
    (1, 4, 2, [4] * 4, [4] * 4),      # Fig 8 {1,4}: K = 256, Local = 2
    (1, 2, 2, [8, 4, 4], [4, 8, 4]),  # mixed, non-square (scalar pull path)
    (1, 2, 2, [2, 16, 16, 16, 8, 8], [2, 16, 16, 16, 8, 8]),      # v9 ends a round with rho = 1: no push
    (1, 2, 2, [2, 16, 16, 8, 8, 4, 4], [2, 16, 16, 8, 8, 4, 4]),  # 3-pass push round (intermediates first)
]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("push", [True, False])
@pytest.mark.parametrize("GM,GK,M,P,Q", GRIDS)
def test_dist_p2p(GM, GK, M, P, Q, push):
    """push=True: non-final rounds whose last pass is the v9 cluster kernel or a v6 fp32 chunk-pair
    kernel store straight into the peers' heaps (the fused exchange); every other round, and every round
    with push=False, goes through the pull kernel."""
    import torch.multiprocessing as mp
    world = GM * GK
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, GM, GK, M, P, Q, q, push)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    res, t0 = [], time.time()
    while len(res) < world and time.time() - t0 < 300:
        try:
            res.append(q.get(timeout=5))
        except queue.Empty:
            if not any(p.is_alive() for p in procs):  # a rank died without reporting: fail fast
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert len(res) == world, f"only {len(res)} of {world} ranks reported (exit codes {[p.exitcode for p in procs]})"
    res.sort()
    for rank, ok, timeouts in res:
        assert all(v is True for v in ok), f"rank {rank}: {ok}"
        assert timeouts == 0, f"rank {rank}: {timeouts} barrier timeouts"
    assert all(p.exitcode == 0 for p in procs)
