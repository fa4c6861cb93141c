"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck):
every path on partial tiles, transposes, stream-K, beta = 0 and alpha = 0,
and the three convolution kernels."""
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
torch.cuda.synchronize()
print("sanitize cases done")
