"""Soaked (power-capped steady state) time of one rank's GEMM at P = 8 / 4
(m = 2048 / 4096, n = k = 16384) per tensor-core configuration, full K and the
geometric K-chunk chain, vs T1/P."""
import os, statistics, sys, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1804_10694_b200 as tm
S = 16384
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.rand(S, S, device="cuda", generator=g); B = torch.rand(S, S, device="cuda", generator=g); C = torch.rand(S, S, device="cuda", generator=g)
def soak_time(fn, seconds=1.5, reps=5):
    t0 = time.time()
    while time.time() - t0 < seconds:
        fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts), 3)
T1 = soak_time(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5))
out = {"T1": T1}
for P in (8, 4):
    r0, rows = tm.dist_rows(S, P, 0)
    Ar, Cr = A[:rows], C[:rows]
    chunks = tm.dist_chunks(S, P)
    for cfg in ("auto", "2,128,0", "2,128,1", "2,64,0", "1,128,0"):
        if cfg != "auto":
            os.environ["TM_TC_CONFIG"] = cfg
        full = soak_time(lambda: tm.sgemm_ex(Ar, B, Cr, 1.5, 0.5))
        chain = soak_time(lambda: [tm.sgemm_ex(Ar[:, k0:k0 + kr], B[k0:k0 + kr], Cr, 1.5, 0.5 if i == 0 else 1.0) for i, (k0, kr) in enumerate(chunks)])
        os.environ.pop("TM_TC_CONFIG", None)
        out[f"P{P}_{cfg}"] = {"full": full, "chain": chain, "eff_full": round(T1 / P / full, 3), "eff_chain": round(T1 / P / chain, 3)}
        print(P, cfg, out[f"P{P}_{cfg}"], flush=True)
print(json.dumps(out))
