import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm
for s in (4096, 8192):
    for opa in "NT":
        for opb in "NT":
            A = torch.rand(s, s, device="cuda"); B = torch.rand(s, s, device="cuda"); C = torch.rand(s, s, device="cuda")
            for _ in range(2): tm.sgemm_op(A, B, C, 1.5, 0.5, opa, opb)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): tm.sgemm_op(A, B, C, 1.5, 0.5, opa, opb)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"{s}^3 {opa}{opb}: {ms:.3f} ms  {2*s**3/ms/1e9:.0f} GFLOP/s", flush=True)
