"""Crossover of the small-GEMM kernel vs the tensor-core kernel (event-timed,
after a 512 MiB read-flush, median of 30): sets the AUTO threshold."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1804_10694_b200 as tm

flush = torch.ones(512 * 2 ** 20 // 4, device="cuda")
fo = torch.empty(1, device="cuda")
tiny = torch.zeros(1, device="cuda")


def t_of(fn, reps=30):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=fo[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    return round(statistics.median(ts), 2)


print("empty launch", t_of(lambda: tiny.add_(1)))
for (m, n, k) in [(64, 64, 64), (128, 128, 128), (192, 192, 192), (256, 256, 256), (320, 320, 320), (384, 384, 384),
                  (512, 512, 512), (768, 768, 768), (1060, 1060, 1060), (4096, 64, 64), (64, 64, 4096), (50176, 64, 64)]:
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    A = torch.rand(m, k, device="cuda", generator=g); B = torch.rand(k, n, device="cuda", generator=g)
    C = torch.rand(m, n, device="cuda", generator=g)
    os.environ["TM_SMALL_MAX"] = str(1 << 62)
    small = t_of(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 0))
    os.environ["TM_SMALL_MAX"] = "0"
    tc = t_of(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 0))
    best = (1e9, None)
    for cfg in ["2,128,0", "2,64,0", "2,64,1", "1,128,0", "1,128,1", "1,64,0", "1,32,0", "1,32,1"]:
        os.environ["TM_TC_CONFIG"] = cfg
        v = t_of(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 1), reps=15)
        best = min(best, (v, cfg))
    del os.environ["TM_TC_CONFIG"]
    del os.environ["TM_SMALL_MAX"]
    print(json.dumps({"mnk": [m, n, k], "macs_log2": round(__import__("math").log2(m * n * k), 2), "small": small,
                      "tc_auto": tc, "tc_best": best}), flush=True)
