"""Row-sharded multi-GPU mode, verified on one GPU through the loopback
(tm_sgemm_dist_loopback): the same partition, K-chunk schedule and beta chain
as tm_sgemm_dist, with each chunk broadcast replaced by a device copy.

Checks (SURVEY.md section 4 "Distribution semantics"): each rank's shard equals
the oracle's rows (rows distributed; no gather);
uneven m % P; P = 1 is bit-identical to tm_sgemm; root != 0; each non-root rank
receives exactly k*ldb*4 bytes (message conservation); the all-gather variant."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _run(P, root, m, n, k, seed, kind="uniform", ldb=None, fused=False, transport="nccl"):
    import torch
    import paper_1804_10694_b200 as tm
    ldb = n if ldb is None else ldb
    A, B, C0 = si.matrices(m, n, k, seed, kind=kind, ldb=ldb)
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    Bfull = np.full((k, ldb), np.nan, dtype=np.float32)
    Bfull[:, :n] = B
    Bs, As, Cs, parts = [], [], [], []
    for r in range(P):
        r0, rows = tm.dist_rows(m, P, r)
        parts.append((r0, rows))
        As.append(dA[r0:r0 + rows])
        Cs.append(torch.from_numpy(np.ascontiguousarray(C0[r0:r0 + rows])).cuda())
        if r == root or transport == "ce":  # the copy-engine model moves no data (tm.h)
            Bs.append(torch.from_numpy(Bfull).cuda())
        else:
            Bs.append(torch.full((k, ldb), float("nan"), dtype=torch.float32, device="cuda"))
    got = tm.sgemm_dist_loopback(m, n, k, As, [b for b in Bs], Cs, si.ALPHA, si.BETA, root=root, fused=fused,
                                 transport=transport)
    torch.cuda.synchronize()
    return A, B, C0, parts, [c.cpu().numpy() for c in Cs], got, [b[:, :n].cpu().numpy() for b in Bs]


@pytest.mark.parametrize("transport", ["nccl", "ce"])
@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("P,root", [(2, 0), (3, 1), (8, 0), (8, 5)])
def test_loopback_shards_match_oracle(P, root, fused, transport):
    """fused=False: K-chunked schedule (beta chain); fused=True: one GEMM per
    rank whose TMA producers wait on per-chunk flags set by the copy stream.
    transport="ce": the copy-engine transport model (every B pre-filled, chunks
    released on the link model's schedule, GEMMs on every SM but one)."""
    m, n, k = 1060, 260, 1100   # uneven rows; two K-chunks of 512 and 588
    A, B, C0, parts, Cs, got, Bs = _run(P, root, m, n, k, seed=40 + P, fused=fused, transport=transport)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    for r, ((r0, rows), C) in enumerate(zip(parts, Cs)):
        assert C.shape == (rows, n)
        if rows:
            e = float(np.max(oracle.normalized_error(C, R[r0:r0 + rows], D[r0:r0 + rows])))
            assert e <= TOL, (r, e)
        assert np.array_equal(Bs[r], B)  # every rank ends with root's B
        assert got[r] == (0 if r == root else k * n * 4)  # message conservation


def test_loopback_p1_bit_identical_to_sgemm():
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 700, 300, 900
    A, B, C0, parts, Cs, got, _ = _run(1, 0, m, n, k, seed=50)
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, B, C0))
    tm.sgemm(dA, dB, dC, si.ALPHA, si.BETA)
    assert np.array_equal(Cs[0], dC.cpu().numpy()) and got == [0]


def test_loopback_more_ranks_than_rows():
    m, n, k = 5, 40, 700
    A, B, C0, parts, Cs, got, _ = _run(8, 0, m, n, k, seed=51)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    assert sum(rows for _, rows in parts) == m
    for (r0, rows), C in zip(parts, Cs):
        if rows:
            assert float(np.max(oracle.normalized_error(C, R[r0:r0 + rows], D[r0:r0 + rows]))) <= TOL


@pytest.mark.parametrize("fused", [False, True])
def test_loopback_c5_p8_sampled_rows(fused):
    """BASELINE.json configs[4]: 16384^3 row-sharded over 8 ranks (geometric
    K-chunks 512 ... 8704; fused: 8 uniform flag chunks of 2048), sampled rows incl. every shard boundary, all-positive stress data
    (the beta chain adds 7 extra fp32 roundings per element)."""
    import torch
    import paper_1804_10694_b200 as tm
    m = n = k = 16384
    P = 8
    A, B, C0 = si.matrices(m, n, k, si.SEEDS["C5"], kind="positive")
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    Bs = [dB] + [torch.empty_like(dB) for _ in range(P - 1)]
    As, Cs, bounds = [], [], []
    for r in range(P):
        r0, rows = tm.dist_rows(m, P, r)
        bounds += [r0, r0 + rows - 1]
        As.append(dA[r0:r0 + rows])
        Cs.append(torch.from_numpy(C0[r0:r0 + rows].copy()).cuda())
    tm.sgemm_dist_loopback(m, n, k, As, Bs, Cs, si.ALPHA, si.BETA, fused=fused)
    C = torch.cat(Cs).cpu().numpy()
    del Bs, dA, dB, As, Cs
    torch.cuda.empty_cache()
    rows = si.sample_rows(m, count=24, tile=2048, extra=bounds)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, rows=rows)
    assert float(np.max(oracle.normalized_error(C[rows], R, D))) <= TOL


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_loopback_allgather_shards_match_oracle(P):
    """All-gather variant: B pre-sharded by k-rows (k % P == 0); each rank's
    GEMM on its own shard overlaps the gather; every rank ends with full B."""
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 1060, 260, 1024
    A, B, C0 = si.matrices(m, n, k, seed=60 + P)
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    kr = k // P
    Bs, As, Cs, parts = [], [], [], []
    for r in range(P):
        r0, rows = tm.dist_rows(m, P, r)
        parts.append((r0, rows))
        As.append(dA[r0:r0 + rows])
        Cs.append(torch.from_numpy(np.ascontiguousarray(C0[r0:r0 + rows])).cuda())
        buf = torch.full((k, n), float("nan"), dtype=torch.float32, device="cuda")
        buf[r * kr:(r + 1) * kr] = torch.from_numpy(B[r * kr:(r + 1) * kr]).cuda()
        Bs.append(buf)
    got = tm.sgemm_dist_loopback(m, n, k, As, Bs, Cs, si.ALPHA, si.BETA, allgather=True)
    torch.cuda.synchronize()
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    for r, ((r0, rows), C) in enumerate(zip(parts, Cs)):
        e = float(np.max(oracle.normalized_error(C.cpu().numpy(), R[r0:r0 + rows], D[r0:r0 + rows])))
        assert e <= TOL, (r, e)
        assert np.array_equal(Bs[r].cpu().numpy(), B)
        assert got[r] == (P - 1) * kr * n * 4


def test_loopback_fused_many_chunks_and_slow_link():
    """Fused mode with 8 chunks, misaligned-free but ragged tiles, and the
    transfer slowed to a modelled 200 GB/s link (TM_LOOPBACK_LINK_GBS): the
    gated GEMM must wait for every chunk and still match the oracle; integer
    inputs bit-exact (one GEMM per rank: no beta chain roundings)."""
    import os
    os.environ["TM_LOOPBACK_LINK_GBS"] = "200"
    try:
        m, n, k = 777, 300, 4100  # 8 chunks of 544 rows, ragged last
        A, B, C0, parts, Cs, got, Bs = _run(4, 2, m, n, k, seed=70, kind="integer", fused=True)
    finally:
        del os.environ["TM_LOOPBACK_LINK_GBS"]
    R, _ = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    for r, ((r0, rows), C) in enumerate(zip(parts, Cs)):
        assert np.array_equal(C.astype(np.float64), R[r0:r0 + rows]), r
        assert got[r] == (0 if r == 2 else k * n * 4)
