"""C3 4096^3 and C2 1060^3 per tensor-core configuration, soaked (power-capped
steady state), median of 20 event-timed runs with the bench's L2 flush."""
import os, statistics, sys, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1804_10694_b200 as tm
flush = torch.ones(512 * 2 ** 20 // 4, device="cuda"); fo = torch.empty(1, device="cuda")
def soak_time(fn, seconds=1.0, reps=20):
    t0 = time.time()
    while time.time() - t0 < seconds:
        torch.sum(flush, dim=0, out=fo[0]); fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=fo[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts) * 1000, 1)
for S in (4096, 1060):
    g = torch.Generator(device="cuda").manual_seed(1)
    A, B, C = (torch.rand(S, S, device="cuda", generator=g) for _ in range(3))
    res = {}
    for cfg in ["auto", "2,128,0", "2,128,1", "2,64,0", "2,64,1", "1,128,0", "1,128,1", "1,64,1"]:
        if cfg != "auto": os.environ["TM_TC_CONFIG"] = cfg
        res[cfg] = soak_time(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5))
        os.environ.pop("TM_TC_CONFIG", None)
    print(S, json.dumps(res), flush=True)
