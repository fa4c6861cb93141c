"""Loopback timing sanity: P = 8, C5; device-event time of the whole loopback
call (all ranks) / P, for the chunked and fused schedules under the NCCL
model (devcopy) and the copy-engine model at an effectively infinite link and
at 700 GB/s, plus the direct per-rank GEMM times."""
import os, statistics, sys, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1804_10694_b200 as tm
S, P = 16384, int(os.environ.get("P", "8"))
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.rand(S, S, device="cuda", generator=g); B = torch.rand(S, S, device="cuda", generator=g); C = torch.rand(S, S, device="cuda", generator=g)
Al, Bl, Cl = [], [], []
for r in range(P):
    r0, rows = tm.dist_rows(S, P, r); Al.append(A[r0:r0 + rows]); Cl.append(C[r0:r0 + rows]); Bl.append(B if r == 0 else B.clone())
def t(fn, reps=3):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - h0) * 1e3))
    return [round(min(x[0] for x in ts) / P, 3), round(min(x[1] for x in ts) / P, 3)]
res = {"rank_gemm_fullK": t(lambda: [tm.sgemm_ex(Al[r], B, Cl[r], 1.5, 0.5) for r in range(P)])}
for tr in ("nccl", "ce"):
    for fused in (False, True):
        for link in ((None,) if tr == "nccl" else ("1000000", "700")):
            if link: os.environ["TM_LOOPBACK_LINK_GBS"] = link
            res[f"{tr}_{'fused' if fused else 'chunked'}_{link}"] = t(lambda: tm.sgemm_dist_loopback(S, S, S, Al, Bl, Cl, 1.5, 0.5, fused=fused, transport=tr))
            os.environ.pop("TM_LOOPBACK_LINK_GBS", None)
print(json.dumps(res))
