"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck):
every path on partial tiles, transposes, stream-K, beta = 0 and alpha = 0,
the precision variants, the small-GEMM kernel, the three convolution kernels
(direct incl. passes of filter rows and the two-launch filter split), the blur
and the loopback distributed schedules (chunked, fused, SUMMA, blur)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm

g = torch.Generator(device="cuda"); g.manual_seed(0)
def t(r, c, ld=None):
    ld = ld or c
    return torch.rand((r, ld), generator=g, device="cuda")[:, :c]
cases = [(64, 64, 64), (300, 260, 200), (129, 65, 33), (1060, 132, 100)]
for (m, n, k) in cases:
    for algo in (1, 2):
        for beta in (0.5, 0.0):
            A, B = t(m, k, (k + 7) // 4 * 4), t(k, n, (n + 3) // 4 * 4)
            C = t(m, n, (n + 3) // 4 * 4 + 4)
            tm.sgemm_ex(A, B, C, 1.5, beta, algo)
        for opa, opb in (("T", "N"), ("N", "T"), ("T", "T")):
            A = t(k, m, (m + 3) // 4 * 4) if opa == "T" else t(m, k, (k + 3) // 4 * 4)
            B = t(n, k, (k + 3) // 4 * 4) if opb == "T" else t(k, n, (n + 3) // 4 * 4)
            C = t(m, n, (n + 3) // 4 * 4)
            tm.sgemm_op(A, B, C, 1.5, 0.5, opa, opb, algo=algo)
    for cfg in ("2,128,1", "1,64,1", "2,32,0"):
        os.environ["TM_TC_CONFIG"] = cfg
        A, B, C = t(m, k, (k + 3) // 4 * 4), t(k, n, (n + 3) // 4 * 4), t(m, n, (n + 3) // 4 * 4)
        tm.sgemm_ex(A, B, C, 1.5, 0.5, 1)
        del os.environ["TM_TC_CONFIG"]
    A, B, C = t(m, k), t(k, n), t(m, n)
    tm.sgemm_ex(A, B, C, 0.0, 0.5, 0)
# hybrid stream-K (more tiles than clusters): partial wave split, then whole tiles
for (m, n, k, cfg) in ((2500, 300, 200, "1,32,1"), (2500, 2100, 300, "2,64,1")):
    os.environ["TM_TC_CONFIG"] = cfg
    A, B, C = t(m, k), t(k, n), t(m, n)
    tm.sgemm_ex(A, B, C, 1.5, 0.5, 1)
    del os.environ["TM_TC_CONFIG"]
# convolution: direct (S in {1, 3}), implicit-GEMM (forced and S = 5), SIMT; ragged rows, beta 0 / 0.5
for (nb, h, w, c, f, r, s, pad) in [(2, 5, 140, 16, 16, 3, 3, 1), (1, 4, 130, 32, 24, 3, 3, 1),
                                     (2, 3, 131, 16, 40, 1, 1, 0), (1, 6, 37, 16, 8, 5, 5, 2),
                                     (1, 5, 20, 48, 20, 3, 3, 1)]:
    ho, wo = h + 2 * pad - r + 1, w + 2 * pad - s + 1
    X, Wt = torch.rand((nb, h, w, c), generator=g, device="cuda"), torch.rand((f, r, s, c), generator=g, device="cuda")
    for path in (None, "im2col"):
        for beta in (0.5, 0.0):
            if path:
                os.environ["TM_CONV_PATH"] = path
            Y = torch.rand((nb, ho, wo, f), generator=g, device="cuda")
            tm.conv2d_nhwc(X, Wt, Y, 1.5, beta, pad)
            os.environ.pop("TM_CONV_PATH", None)
    Y = torch.rand((nb, ho, wo, f), generator=g, device="cuda")
    tm.conv2d_nhwc(X, Wt, Y, 1.5, 0.5, pad, algo=2)
# round 2: precision variants, small-GEMM kernel, wide filters, blur, loopback schedules
for algo in (3, 4):
    A, B, C = t(300, 200, 200), t(200, 260, 260), t(300, 260, 260)
    tm.sgemm_ex(A, B, C, 1.5, 0.5, algo)
A, B, C = t(50, 60), t(60, 70), t(50, 70)
tm.sgemm_ex(A, B, C, 1.5, 0.5, 0)  # small-GEMM kernel
for (nb, h, w, c, f, r, s, pad) in [(1, 12, 60, 16, 16, 7, 7, 3), (1, 14, 50, 16, 16, 9, 9, 4),
                                     (1, 15, 40, 16, 16, 11, 11, 5)]:
    ho, wo = h + 2 * pad - r + 1, w + 2 * pad - s + 1
    X, Wt = torch.rand((nb, h, w, c), generator=g, device="cuda"), torch.rand((f, r, s, c), generator=g, device="cuda")
    Y = torch.rand((nb, ho, wo, f), generator=g, device="cuda")
    tm.conv2d_nhwc(X, Wt, Y, 1.5, 0.5, pad)
for (N, M) in [(3, 3), (37, 41), (130, 301)]:
    img = torch.rand((N, M, 3), generator=g, device="cuda")
    tm.blur(img)
    if M > 3:
        tm.blur(img[:, 1:, :])  # padded pitch, offset base
P, N, M = 3, 40, 33
lins, louts = [], []
for r in range(P):
    rows = tm.dist_rows(N - 2, P, r)[1]
    lins.append(torch.rand((rows + 2, M, 3), generator=g, device="cuda"))
    louts.append(torch.empty((rows, M - 2, 3), device="cuda"))
tm.blur_dist_loopback(N, M, lins, louts)
m, n, k = 300, 260, 1100
A, B = t(m, k), t(k, n)
for fused in (False, True):
    As = [A[r0:r0 + rows] for r0, rows in (tm.dist_rows(m, 3, r) for r in range(3))]
    Cs = [t(rows, n) for _, rows in (tm.dist_rows(m, 3, r) for r in range(3))]
    Bs = [B.contiguous()] + [torch.empty((k, n), device="cuda") for _ in range(2)]
    tm.sgemm_dist_loopback(m, n, k, As, Bs, [c.contiguous() for c in Cs], 1.5, 0.5, fused=fused)
pr, pc = 2, 2
As, Bs, Cs = [], [], []
for r in range(pr * pc):
    (r0, rows), (c0, cols), (a0, ka), (b0, kb) = tm.summa_blocks(m, n, k, pr, pc, r)
    As.append(t(rows, ka).contiguous()); Bs.append(t(kb, cols).contiguous()); Cs.append(t(rows, cols).contiguous())
tm.sgemm_summa_loopback(pr, pc, m, n, k, As, Bs, Cs, 1.5, 0.5)
torch.cuda.synchronize()
print("sanitize cases done")
