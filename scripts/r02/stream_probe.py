"""C4-sized streaming references (event-timed medians, L2 flushed): a plain
read of A (50176 x 576 fp32) and a read+write of A, beside the C4 GEMM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1804_10694_b200 as tm
flush = torch.ones(512 * 2 ** 20 // 4, device="cuda"); fo = torch.empty(1, device="cuda")
m, n, k = 50176, 64, 576
A = torch.rand(m, k, device="cuda"); B = torch.rand(k, n, device="cuda"); C = torch.rand(m, n, device="cuda")
D = torch.empty_like(A); r = torch.empty(m, device="cuda")


def timed(fn, reps=50):
    out = []
    for _ in range(reps + 5):
        torch.sum(flush, dim=0, out=fo[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3)
    out = sorted(out[5:])
    return out[len(out) // 2]


lib = os.environ.get("TM_LIB_PATH", "product")
for name, fn, nbytes in (("read A (sum rows)", lambda: torch.sum(A, dim=1, out=r), A.numel() * 4),
                         ("copy A", lambda: D.copy_(A), 2 * A.numel() * 4),
                         ("C4 sgemm", lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 1), (m * k + k * n + 2 * m * n) * 4)):
    t = timed(fn)
    print(f"{lib}: {name:18s} {t:7.2f} us  {nbytes / t / 1e6:6.2f} TB/s", flush=True)
