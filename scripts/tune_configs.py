"""Tune the BASELINE.json GEMM configs (tm_sgemm_tune) and compare the tuned
choice with the cost-model plan: median device time of each over 20 runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10694_b200 as tm

flush = torch.ones(512 * 2**20 // 4, device="cuda"); out = torch.empty(1, device="cuda")


def t(fn, reps=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=out[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort(); return ts[len(ts) // 2]


for name, (m, n, k) in [("C2", (1060, 1060, 1060)), ("C4", (50176, 64, 576)), ("C3", (4096, 4096, 4096)),
                        ("odd", (3000, 700, 2500)), ("skinny", (20000, 128, 4096))]:
    A = torch.rand(m, k, device="cuda"); B = torch.rand(k, n, device="cuda"); C = torch.rand(m, n, device="cuda")
    tm.tune_cache_clear()
    plan = tm.plan_config(m, n, k, 1.5, 0.5, A.data_ptr(), k, B.data_ptr(), n, C.data_ptr(), n)
    t0 = t(lambda: tm.sgemm(A, B, C, 1.5, 0.5))
    cg, bn, sk, ms = tm.tune(A, B, C, 1.5, 0.5, reps=5)
    t1 = t(lambda: tm.sgemm(A, B, C, 1.5, 0.5))
    print(f"{name} {m}x{n}x{k}: model plan cg={plan[1]} bn={plan[2]} sk={plan[3]} {t0:.1f} us | "
          f"tuned cg={cg} bn={bn} sk={sk} {t1:.1f} us ({(t0 / t1 - 1) * 100:+.1f}%)", flush=True)
