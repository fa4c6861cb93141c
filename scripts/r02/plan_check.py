"""Planner vs every tensor-core configuration (with the hybrid stream-K schedule)
on mid-size shapes: soaked event-timed medians, L2 flushed for shapes that fit."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1804_10694_b200 as tm
flush = torch.ones(512 * 2 ** 20 // 4, device="cuda"); fo = torch.empty(1, device="cuda")


def timed(fn, reps=15):
    t0 = time.time()
    while time.time() - t0 < 0.5:
        fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=fo[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for (m, n, k) in ((4096, 4096, 4096), (3000, 3000, 3000), (6000, 6000, 2000), (2048, 8192, 4096), (12000, 1000, 3000)):
    A = torch.rand(m, k, device="cuda"); B = torch.rand(k, n, device="cuda"); C = torch.rand(m, n, device="cuda")
    res = {}
    for cfg in ("auto", "2,128,0", "2,128,1", "2,64,0", "2,64,1", "1,128,0", "1,128,1"):
        if cfg != "auto":
            os.environ["TM_TC_CONFIG"] = cfg
        else:
            os.environ.pop("TM_TC_CONFIG", None)
        ms = timed(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 1))
        res[cfg] = round(2 * m * n * k / ms / 1e9, 1)
    os.environ.pop("TM_TC_CONFIG", None)
    best = max((v, c) for c, v in res.items() if c != "auto")
    print(f"{m}x{n}x{k}: auto {res['auto']} TFLOP/s ({tm.plan_config(m, n, k)}), best {best[1]} {best[0]}; {res}", flush=True)
