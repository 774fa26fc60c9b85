"""Debug the tcgen05 pair kernel on structured inputs (identity / one-hot factors) against the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
from paper_2401_10187_b200 import kron

dev = torch.device("cuda:0")
rng = np.random.default_rng(1)
for P in (32, 16):
    R = 8 if P == 32 else 16
    M, K = 1, P * P * R
    nF = 2 if P == 32 else 2
    for mode in ("tf32", "3xtf32"):
        for name, F1, F2 in (("I,I", np.eye(P), np.eye(P)),
                             ("I,rand", np.eye(P), rng.integers(-1, 2, (P, P)).astype(float)),
                             ("rand,I", rng.integers(-1, 2, (P, P)).astype(float), np.eye(P)),
                             ("rand,rand", rng.integers(-1, 2, (P, P)).astype(float), rng.integers(-1, 2, (P, P)).astype(float))):
            X = (np.arange(M * K) % 7 - 3).reshape(M, K).astype(np.float32)
            # F^1 = I_R (applied last, CUDA cores, exact), F^2 = F2 (second), F^3 = F1 (first): the pair pass sees
            # rows of R chunks
            Fs = [np.eye(R, dtype=np.float32), F2.astype(np.float32), F1.astype(np.float32)]
            ref = oracle.alg1(X, Fs).astype(np.float32)
            Y = kron.matmul(torch.from_numpy(X).to(dev), [torch.from_numpy(f).to(dev) for f in Fs], mode=mode)
            torch.cuda.synchronize()
            Y = Y.cpu().numpy()
            bad = np.argwhere(Y != ref)
            print(P, mode, name, kron.plan_kernels(M, [R, P, P], [R, P, P], "float32", mode), "mismatches", len(bad), "of", Y.size,
                  "first", bad[:3].tolist(), Y.ravel()[:6], ref.ravel()[:6], flush=True)
            if len(bad) and name == "I,I":
                # where did each output come from?  X values are small ints; print a map of Y vs X
                print("   Y[:40]", Y.ravel()[:40].tolist())
                print("   X[:40]", X.ravel()[:40].tolist())
