"""Bring-up diagnostics for the tcgen05 path: structured inputs whose products
reveal row/column/K mappings.  Prints compact summaries."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm  # noqa: E402

np.set_printoptions(linewidth=200, precision=3, suppress=True)


def gemm(A, B, algo=3, config=None):
    if config:
        os.environ["TM_TC_CONFIG"] = config
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    dC = torch.zeros((A.shape[0], B.shape[1]), dtype=torch.float32, device="cuda")
    tm.sgemm_ex(dA, dB, dC, 1.0, 0.0, algo)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


def show(name, C, E):
    ok = np.isclose(C, E, rtol=1e-2, atol=1e-3)
    print(f"--- {name}: {ok.mean()*100:.1f}% ok, nonzero {np.count_nonzero(C)}/{C.size}")
    if not ok.all():
        print("C[:4,:16]=\n", C[:4, :16])
        print("E[:4,:16]=\n", E[:4, :16])
        bad = np.argwhere(~ok)
        print("first bad:", bad[:8].tolist())
        rows_ok = ok.all(axis=1)
        cols_ok = ok.all(axis=0)
        print("rows ok:", np.flatnonzero(rows_ok)[:20], "... count", rows_ok.sum())
        print("cols ok:", np.flatnonzero(cols_ok)[:40], "... count", cols_ok.sum())


for config in sys.argv[1:] or ["1,32", "1,128", "2,32", "2,128"]:
    cg, bn = (int(x) for x in config.split(","))
    M, N = 128 * cg, bn * cg
    print(f"===================== config {config}: tile {M}x{N}")
    for K in (8, 32, 64):
        # (1) B row 0 = j+1, A col 0 = 1  ->  C[i,j] = j+1
        A = np.zeros((M, K), np.float32); A[:, 0] = 1
        B = np.zeros((K, N), np.float32); B[0, :] = np.arange(N) + 1
        show(f"K={K} colmap", gemm(A, B, config=config), A @ B)
        # (2) A col 0 = i+1, B row 0 = 1  ->  C[i,j] = i+1
        A = np.zeros((M, K), np.float32); A[:, 0] = np.arange(M) + 1
        B = np.zeros((K, N), np.float32); B[0, :] = 1
        show(f"K={K} rowmap", gemm(A, B, config=config), A @ B)
        # (3) K mapping: A[i,p] = p+1, B[p,j] = 1 if p == j % K
        A = np.tile(np.arange(K, dtype=np.float32) + 1, (M, 1))
        B = np.zeros((K, N), np.float32)
        for j in range(N):
            B[j % K, j] = 1
        show(f"K={K} kmap", gemm(A, B, config=config), A @ B)
        # (4) random, small integers
        g = np.random.default_rng(K)
        A = g.integers(-3, 4, (M, K)).astype(np.float32)
        B = g.integers(-3, 4, (K, N)).astype(np.float32)
        show(f"K={K} random-int", gemm(A, B, config=config), A @ B)
