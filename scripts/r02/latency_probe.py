"""Event-timed latency breakdown for the small configs (C1 64^3, C2 1060^3):
floor of an empty launch, every tensor-core config, SIMT; same harness as
bench.py (512 MiB read-flush, then events around the call). Median of 30."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1804_10694_b200 as tm

flush = torch.ones(512 * 2 ** 20 // 4, device="cuda")
fo = torch.empty(1, device="cuda")
tiny = torch.zeros(1, device="cuda")


def t_of(fn, reps=30, do_flush=True):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if do_flush:
            torch.sum(flush, dim=0, out=fo[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    return round(statistics.median(ts), 2)


print("empty launch (tiny.add_)", t_of(lambda: tiny.add_(1)))
for s in [64, 128, 256, 512, 1060, 2048]:
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    A, B, C = (torch.rand(s, s, device="cuda", generator=g) for _ in range(3))
    res = {"simt": t_of(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 2)), "auto": t_of(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 0))}
    for cfg in ["2,128,0", "2,128,1", "2,64,0", "2,64,1", "1,128,0", "1,128,1", "1,64,0", "1,64,1", "1,32,0", "1,32,1"]:
        os.environ["TM_TC_CONFIG"] = cfg
        try:
            res[cfg] = t_of(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 1))
        except Exception as e:
            res[cfg] = str(e)[:40]
        del os.environ["TM_TC_CONFIG"]
    print(s, json.dumps(res), flush=True)
