import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm
for s in [64, 96, 128, 192, 256, 384, 512, 768]:
    A = torch.rand(s, s, device="cuda"); B = torch.rand(s, s, device="cuda"); C = torch.rand(s, s, device="cuda")
    res = {}
    for name, algo in [("tc", 1), ("simt", 2)]:
        for _ in range(3): tm.sgemm_ex(A, B, C, 1.5, 0.5, algo)
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); tm.sgemm_ex(A, B, C, 1.5, 0.5, algo); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        ts.sort(); res[name] = round(ts[10], 2)
    print(s, res, flush=True)
