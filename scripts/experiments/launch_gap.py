"""How much of a small GEMM's event time is the flush->GEMM transition?
Event time per call with the bench's L2 flush before each call vs back to back."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1804_10694_b200 as tm

flush = torch.ones(512 * 2**20 // 4, device="cuda"); out = torch.empty(1, device="cuda")

def ev_time(fn, reps=20, pre=None):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        if pre: pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort(); return round(ts[len(ts) // 2], 1)

def b2b(fn, reps=50):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1000 / reps, 1)

fl = lambda: torch.sum(flush, dim=0, out=out[0])
for (m, n, k) in [(64, 64, 64), (1060, 1060, 1060), (50176, 64, 576), (4096, 4096, 4096)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.rand(m, k, device="cuda", generator=g) * 2 - 1
    B = torch.rand(k, n, device="cuda", generator=g) * 2 - 1
    C = torch.rand(m, n, device="cuda", generator=g) * 2 - 1
    f = lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, tm.ALGO_TF32X3)
    print(f"{m}x{n}x{k}: flushed {ev_time(f, pre=fl)} us, no flush {ev_time(f)} us, back-to-back {b2b(f)} us/call")
x = torch.empty(1, device="cuda")
print("tiny torch kernel after flush", ev_time(lambda: x.add_(1), pre=fl), "b2b", b2b(lambda: x.add_(1)))
A = torch.rand(50176, 576, device="cuda"); D = torch.empty_like(A)
print("C4 A copy (2x115.6 MB) after flush", ev_time(lambda: D.copy_(A), pre=fl), "us")
print("C4 A sum after flush", ev_time(lambda: torch.sum(A, dim=0), pre=fl), "us")
