"""Projection of the row-sharded C5 scaling from single-GPU
measurements; NOT a multi-GPU measurement.

Measured on this GPU (CUDA events, median of 5, each after >= 1 s of the same
work back to back so all are taken at the sustained power-capped clock): T1 = one tm_sgemm of the whole
16384^3 problem, and for each P the rank's GEMMs on its K-chunks (geometric
chunk plan, tm_dist_chunk; beta chain) enqueued back to back as the schedule
does, an event after each (g_c = the interval ending at chunk c's event), with
every SM and with the 16 SMs the NCCL schedule leaves to NCCL's kernels
(TM_SM_RESERVE=16).

Modelled: chunk c of B reaches the LAST rank of a pipelined chain (or NCCL
ring) at  a_c = L + ((P-1) * piece + bytes of chunks 0..c) / R  (piece = 128
K-rows as tm_sgemm_dist_ce forwards them, L = 10 us start latency), for link rates R = 700 and 450 GB/s.  The
rank's time is the chunked schedule's  t = 0; for c: t = max(t, a_c) + g_c.
  nccl: g_c with 16 SMs reserved while the broadcast is still running
        (a_last > t at the chunk's start), all SMs afterwards;
  ce:   g_c with every SM (copy engines move B; tm_sgemm_dist_ce).
Efficiency = T1 / (P * T_rank).  Not modelled: the incoming B's HBM writes
(1 GiB per rank over the transfer, ~0.15 ms of HBM time), NCCL's own
efficiency, eight GPUs' power and clocks."""
import json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm

S = int(os.environ.get("S", "16384"))
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.rand(S, S, device="cuda", generator=g) * 2 - 1
B = torch.rand(S, S, device="cuda", generator=g) * 2 - 1
C = torch.rand(S, S, device="cuda", generator=g) * 2 - 1


def soak(fn, seconds=1.0):
    """Run fn back to back for ~seconds so every timing is taken in the same
    sustained (power-capped) clock state as T1."""
    import time
    t0 = time.time()
    while time.time() - t0 < seconds:
        fn()
        torch.cuda.synchronize()


def ev(fn, reps=5):
    soak(fn)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


T1 = ev(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5))
PIECE, L = 128, 0.010


def chain_times(Ar, Cr, chunks, reps=5):
    """Per-chunk GEMM times of the back-to-back chunk chain (median over reps)."""
    def once():
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(chunks) + 1)]
        evs[0].record()
        for i, (k0, kr) in enumerate(chunks):
            tm.sgemm_ex(Ar[:, k0:k0 + kr], B[k0:k0 + kr], Cr, 1.5, 0.5 if i == 0 else 1.0)
            evs[i + 1].record()
        torch.cuda.synchronize()
        return [evs[i].elapsed_time(evs[i + 1]) for i in range(len(chunks))]
    soak(once)
    runs = [once() for _ in range(reps)]
    return [statistics.median(r[i] for r in runs) for i in range(len(chunks))]
out = {"workload": f"sgemm {S}^3 row-sharded, B broadcast (projection from single-GPU chunk timings)",
       "T1_ms": round(T1, 3), "model": __doc__.split("Modelled:")[1].split("Efficiency")[0].strip(), "P": {}}
for P in (2, 4, 8):
    r0, rows = tm.dist_rows(S, P, P - 1)
    Ar, Cr = A[r0:r0 + rows], C[r0:r0 + rows]
    chunks = tm.dist_chunks(S, P)
    g_all = chain_times(Ar, Cr, chunks)
    os.environ["TM_SM_RESERVE"] = "16"
    g_res = chain_times(Ar, Cr, chunks)
    os.environ.pop("TM_SM_RESERVE", None)
    full = ev(lambda: tm.sgemm_ex(Ar, B, Cr, 1.5, 0.5))
    res = {"chunks": chunks, "gemm_ms_all_sms": [round(x, 3) for x in g_all],
           "gemm_ms_16_reserved": [round(x, 3) for x in g_res], "rank_gemm_full_k_ms": round(full, 3),
           "chunked_no_transfer_efficiency": round(T1 / (P * sum(g_all)), 3)}
    for R in (700.0, 450.0):
        row_bytes = 4.0 * S
        arr, cum = [], 0.0
        for k0, kr in chunks:
            cum += kr * row_bytes
            arr.append(L + ((P - 1) * PIECE * row_bytes + cum) / (R * 1e9) * 1e3)
        for transport in ("nccl", "ce"):
            t = 0.0
            for c in range(len(chunks)):
                t = max(t, arr[c])
                busy = transport == "nccl" and arr[-1] > t
                t += g_res[c] if busy else g_all[c]
            res[f"{transport}_chunked_R{int(R)}"] = {"T_rank_ms": round(t, 3),
                                                     "projected_efficiency": round(T1 / (P * t), 3)}
    out["P"][P] = res
    print(P, json.dumps({k: v for k, v in res.items() if k not in ("chunks",)}), flush=True)
print(json.dumps(out))
