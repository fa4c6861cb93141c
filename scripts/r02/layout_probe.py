"""C2 (1060^3) and C4 per operand layout (NN: B as 2 x 32-column MN-major TMA
boxes per stage; NT: B^T one K-major box): does the number of TMA loads per
stage move the small-GEMM time?  Event-timed medians, L2 flushed (512 MiB read)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1804_10694_b200 as tm
flush = torch.ones(512 * 2 ** 20 // 4, device="cuda"); fo = torch.empty(1, device="cuda")


def timed(fn, reps=50):
    out = []
    for _ in range(reps + 5):
        torch.sum(flush, dim=0, out=fo[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3)
    out = sorted(out[5:])
    return out[len(out) // 2]


for (m, n, k) in ((1060, 1060, 1060), (1024, 1024, 1024), (50176, 64, 576)):
    A = torch.rand(m, k, device="cuda"); B = torch.rand(k, n, device="cuda"); Bt = B.t().contiguous()
    At = A.t().contiguous(); C = torch.rand(m, n, device="cuda")
    for name, fn in (("NN", lambda: tm.sgemm_op(A, B, C, 1.5, 0.5, "N", "N")),
                     ("NT", lambda: tm.sgemm_op(A, Bt, C, 1.5, 0.5, "N", "T")),
                     ("TN", lambda: tm.sgemm_op(At, B, C, 1.5, 0.5, "T", "N")),
                     ("TT", lambda: tm.sgemm_op(At, Bt, C, 1.5, 0.5, "T", "T"))):
        print(f"{m}x{n}x{k} {name}: {timed(fn):7.2f} us", flush=True)
