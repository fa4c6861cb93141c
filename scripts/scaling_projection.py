"""Single-GPU projection of the row-sharded C5 scaling; NOT a
multi-GPU measurement.  Both schedules (chunked beta chain, and the fused
flag-gated single launch) and two transports: the on-device copy as is, and
the copy followed by a modelled link of LINK_GBS (default 700 GB/s, env
TM_LOOPBACK_LINK_GBS in the library; conservative: the copy time adds on).

tm_sgemm_dist_loopback runs every rank's schedule of tm_sgemm_dist one after
another on this GPU: the same K-chunked GEMMs (beta for chunk 0, then 1) on
SMs - 16 SMs, gated by per-chunk events, while the B chunks arrive through a
concurrent device-to-device copy on a copy stream (copy engines, no SMs)
standing in for the NCCL broadcast.  One rank's wall time ~ total / P (every
rank has the same rows; the root skips its copies).  Projected efficiency =
T1 / (P * T_rank) with T1 = one tm_sgemm of the whole problem.  What it
cannot show: NVLink bandwidth and NCCL kernels sharing the reserved SMs."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm

S = int(os.environ.get("S", "16384"))
m = n = k = S
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.rand(m, k, device="cuda", generator=g) * 2 - 1
B = torch.rand(k, n, device="cuda", generator=g) * 2 - 1
C = torch.rand(m, n, device="cuda", generator=g) * 2 - 1

def t_one(reps=5):
    for _ in range(2): tm.sgemm_ex(A, B, C, 1.5, 0.5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): tm.sgemm_ex(A, B, C, 1.5, 0.5)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

T1 = t_one()
LINK = float(os.environ.get("LINK_GBS", "700"))
out = {"workload": f"sgemm {S}^3 row-sharded, B broadcast (loopback projection)", "T1_ms": round(T1, 3),
       "link_model_gbs": LINK, "P": {}}
for P in (2, 4, 8):
    Al, Bl, Cl = [], [], []
    for r in range(P):
        r0, rows = tm.dist_rows(m, P, r)
        Al.append(A[r0:r0 + rows]); Cl.append(C[r0:r0 + rows])
        Bl.append(B if r == 0 else torch.empty_like(B))
    res = {}
    for fused in (False, True):
        for link in (0.0, LINK):
            if link:
                os.environ["TM_LOOPBACK_LINK_GBS"] = str(link)
            tm.sgemm_dist_loopback(m, n, k, Al, Bl, Cl, 1.5, 0.5, fused=fused)  # warm-up
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                tm.sgemm_dist_loopback(m, n, k, Al, Bl, Cl, 1.5, 0.5, fused=fused)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) * 1e3)
            os.environ.pop("TM_LOOPBACK_LINK_GBS", None)
            T_rank = min(ts) / P
            key = ("fused" if fused else "chunked") + ("_link%d" % link if link else "_devcopy")
            res[key] = {"T_rank_ms": round(T_rank, 3), "projected_efficiency": round(T1 / (P * T_rank), 3),
                        "projected_gflops": round(2.0 * m * n * k / (T_rank * 1e-3) / 1e9, 1)}
    out["P"][P] = res
    print(P, json.dumps(res), flush=True)
    del Bl
    torch.cuda.empty_cache()
print(json.dumps(out))
