"""C2-shaped epilogue probe: timeline + event time at beta 0 / 0.5 (L2 flushed)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1804_10694_b200 as tm
flush = torch.ones(512 * 2**20 // 4, device="cuda"); out = torch.empty(1, device="cuda")
m = n = k = int(os.environ.get("S", "1060"))
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.rand(m, k, device="cuda", generator=g); B = torch.rand(k, n, device="cuda", generator=g)
C = torch.rand(m, n, device="cuda", generator=g)
for beta in (0.0, 0.5):
    ts = []
    for i in range(23):
        torch.sum(flush, dim=0, out=out[0])
        if i == 22: os.environ["TM_TRACE_PATH"] = f"gpurun_out/trace_epi_b{beta}.jsonl"
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); tm.sgemm_ex(A, B, C, 1.5, beta, 1); e1.record(); torch.cuda.synchronize()
        os.environ.pop("TM_TRACE_PATH", None)
        if i >= 3: ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort(); print("beta", beta, "median us", round(ts[len(ts)//2], 1))
