"""Where a rank's time goes in the row-sharded C5 at P ranks (single GPU):
(a) the rank's GEMM over the full K, (b) the same as K-chunk GEMMs with the
beta chain (geometric / uniform chunks), no transfers, (c) the loopback
schedule (chunk copies on a second stream, SM reservation) per rank."""
import json, os, statistics, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1804_10694_b200 as tm

S = 16384
P = int(os.environ.get("P", "8"))
g = torch.Generator(device="cuda").manual_seed(5)
r0, rows = tm.dist_rows(S, P, 1)
A = torch.rand(rows, S, device="cuda", generator=g) * 2 - 1
B = torch.rand(S, S, device="cuda", generator=g) * 2 - 1
C = torch.rand(rows, S, device="cuda", generator=g) * 2 - 1


def ev_time(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts), 3)


def chunked(bounds):
    def f():
        for i, (k0, kr) in enumerate(bounds):
            tm.sgemm_ex(A[:, k0:k0 + kr], B[k0:k0 + kr], C, 1.5, 0.5 if i == 0 else 1.0)
    return f


out = {"P": P, "rows": rows}
out["full_k_ms"] = ev_time(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5))
geo = tm.dist_chunks(S, P)
uni = [(i * 2048, 2048) for i in range(8)]
out["chunked_geometric_ms"] = ev_time(chunked(geo))
out["chunked_uniform8_ms"] = ev_time(chunked(uni))
out["chunks_geometric"] = geo
T1 = S ** 3 * 2 / 1e9  # GFLOP
print(json.dumps(out), flush=True)
