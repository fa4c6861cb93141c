"""The NCCL data plane of the distributed modes (tm_comm_*, tm_sgemm_dist,
tm_sgemm_dist_fused, tm_sgemm_dist_allgather, tm_sgemm_summa, tm_blur_dist) on
real devices.

* One rank on the single GPU every box has: tm_comm_init (dlopen of libnccl and
  ncclCommInitRankConfig with the hand-declared ncclConfig_t), tm_comm_check,
  tm_comm_bytes_received, Comm.sgemm / Comm.sgemm_allgather at P = 1 against the
  oracle (P = 1 is exactly tm_sgemm: bit-identical), then tm_comm_destroy.
* torch.cuda.device_count() NCCL ranks (skipped below 2 GPUs): tm_sgemm_dist with
  uneven m and root != 0, and the all-gather variant; every rank's shard against
  the oracle's rows at the north_star 1e-5 (PAPER.md:897 rows distributed; no
  gather of C), non-root ranks receive exactly k*ldb*4 bytes
  (message conservation).
"""
import os
import socket
import sys

import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-5


def _err(C, R, D):
    return float(np.max(oracle.normalized_error(C, R, D))) if C.size else 0.0


def test_one_rank_comm_lifecycle_and_sgemm():
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 700, 260, 900
    A, B, C0 = si.matrices(m, n, k, seed=61)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    comm = tm.Comm(0, 1)
    try:
        assert comm.check()
        assert comm.bytes_received() == 0
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        dC = torch.from_numpy(C0).cuda()
        comm.sgemm(m, n, k, dA, dB, dC, si.ALPHA, si.BETA, root=0)
        dCf = torch.from_numpy(C0).cuda()
        comm.sgemm(m, n, k, dA, dB, dCf, si.ALPHA, si.BETA, root=0, fused=True)
        ref = torch.from_numpy(C0).cuda()
        tm.sgemm(dA, dB, ref, si.ALPHA, si.BETA)
        torch.cuda.synchronize()
        assert _err(dC.cpu().numpy(), R, D) <= TOL
        assert torch.equal(dC, ref) and torch.equal(dCf, ref)  # P = 1 is exactly tm_sgemm
        # all-gather variant at P = 1: the one shard is all of B (ncclAllGather
        # copies it into B_full), then the GEMM
        B_full = torch.full((k, n), float("nan"), device="cuda")
        dC2 = torch.from_numpy(C0).cuda()
        comm.sgemm_allgather(m, n, k, dA, dB, B_full, dC2, si.ALPHA, si.BETA)
        torch.cuda.synchronize()
        assert torch.equal(B_full, dB)
        assert _err(dC2.cpu().numpy(), R, D) <= TOL
        assert comm.bytes_received() == 0  # nothing arrives from other ranks
        # 2-D SUMMA on a 1 x 1 grid is tm_sgemm
        dCs = torch.from_numpy(C0).cuda()
        comm.sgemm_summa(1, 1, m, n, k, dA, dB, dCs, si.ALPHA, si.BETA)
        torch.cuda.synchronize()
        assert torch.equal(dCs, ref)
        # the row-distributed blur at P = 1 is tm_blur on the whole image
        N, M = 67, 45
        img = si.image(N, M, seed=64)
        lin = torch.from_numpy(img).cuda()
        lout = torch.full((N - 2, M - 2, 3), float("nan"), device="cuda")
        comm.blur(N, M, lin, lout)
        ref = tm.blur(lin)
        torch.cuda.synchronize()
        assert torch.equal(lout, ref)
        assert comm.bytes_received() == 0
        assert comm.check()
    finally:
        comm.close()
    assert comm.handle is None


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_1804_10694_b200 as tm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # bootstrap only; data moves over NCCL
    out = {}
    try:
        comm = tm.Comm(rank, world)
        # broadcast of B from root = world - 1, uneven rows
        m, n, k, root = 1061, 300, 1100, world - 1
        A, B, C0 = si.matrices(m, n, k, seed=62)
        r0, rows = tm.dist_rows(m, world, rank)
        dA = torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda()
        dC = torch.from_numpy(np.ascontiguousarray(C0[r0:r0 + rows])).cuda()
        dB = torch.from_numpy(B).cuda() if rank == root else torch.full((k, n), float("nan"), device="cuda")
        comm.sgemm(m, n, k, dA, dB, dC, si.ALPHA, si.BETA, root=root)
        torch.cuda.synchronize()
        R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, rows=np.arange(r0, r0 + rows))
        out["bcast_err"] = _err(dC.cpu().numpy(), R, D)
        out["bcast_B_equal"] = bool(np.array_equal(dB.cpu().numpy(), B))
        out["bcast_bytes"] = comm.bytes_received()
        out["bcast_bytes_expected"] = 0 if rank == root else k * n * 4
        # fused single launch (flag-gated GEMM), root 0, same data
        dCf = torch.from_numpy(np.ascontiguousarray(C0[r0:r0 + rows])).cuda()
        dBf = torch.from_numpy(B).cuda() if rank == 0 else torch.full((k, n), float("nan"), device="cuda")
        comm.sgemm(m, n, k, dA, dBf, dCf, si.ALPHA, si.BETA, root=0, fused=True)
        torch.cuda.synchronize()
        out["fused_err"] = _err(dCf.cpu().numpy(), R, D)
        out["fused_B_equal"] = bool(np.array_equal(dBf.cpu().numpy(), B))
        # all-gather variant: rank r holds k-rows [r*k/P, (r+1)*k/P) of B
        k2 = 256 * world
        A2, B2, C2 = si.matrices(m, n, k2, seed=63)
        kr = k2 // world
        shard = torch.from_numpy(np.ascontiguousarray(B2[rank * kr:(rank + 1) * kr])).cuda()
        B_full = torch.full((k2, n), float("nan"), device="cuda")
        dA2 = torch.from_numpy(np.ascontiguousarray(A2[r0:r0 + rows])).cuda()
        dC2 = torch.from_numpy(np.ascontiguousarray(C2[r0:r0 + rows])).cuda()
        before = comm.bytes_received()
        comm.sgemm_allgather(m, n, k2, dA2, shard, B_full, dC2, si.ALPHA, si.BETA)
        torch.cuda.synchronize()
        R2, D2 = oracle.sgemm(si.ALPHA, A2, B2, si.BETA, C2, rows=np.arange(r0, r0 + rows))
        out["ag_err"] = _err(dC2.cpu().numpy(), R2, D2)
        out["ag_B_equal"] = bool(np.array_equal(B_full.cpu().numpy(), B2))
        out["ag_bytes"] = comm.bytes_received() - before
        out["ag_bytes_expected"] = (world - 1) * kr * n * 4
        # 2-D SUMMA: pr x pc grid (2 x world/2 when even), panels broadcast along rows / columns
        pr = 2 if world % 2 == 0 else 1
        pc = world // pr
        m3, n3, k3 = 1030, 700, 2600
        A3, B3, C3 = si.matrices(m3, n3, k3, seed=67)
        (sr0, srows), (sc0, scols), (sa0, ska), (sb0, skb) = tm.summa_blocks(m3, n3, k3, pr, pc, rank)
        dA3 = torch.from_numpy(np.ascontiguousarray(A3[sr0:sr0 + srows, sa0:sa0 + ska])).cuda()
        dB3 = torch.from_numpy(np.ascontiguousarray(B3[sb0:sb0 + skb, sc0:sc0 + scols])).cuda()
        dC3 = torch.from_numpy(np.ascontiguousarray(C3[sr0:sr0 + srows, sc0:sc0 + scols])).cuda()
        comm.sgemm_summa(pr, pc, m3, n3, k3, dA3, dB3, dC3, si.ALPHA, si.BETA)
        torch.cuda.synchronize()
        R3, D3 = oracle.sgemm(si.ALPHA, A3, B3, si.BETA, C3, rows=np.arange(sr0, sr0 + srows))
        out["summa_err"] = _err(dC3.cpu().numpy(), R3[:, sc0:sc0 + scols], D3[:, sc0:sc0 + scols])
        # row-distributed blur: border rows from rank + 1 over NCCL
        N, M = 2112, 3520 // 8
        img = si.image(N, M, seed=65)
        b0, brows = tm.dist_rows(N - 2, world, rank)
        lin = torch.full((brows + 2, M, 3), float("nan"), device="cuda")
        lin[:brows] = torch.from_numpy(img[b0:b0 + brows]).cuda()
        if rank == world - 1:
            lin[brows:] = torch.from_numpy(img[N - 2:]).cuda()
        lout = torch.full((brows, M - 2, 3), float("nan"), device="cuda")
        before = comm.bytes_received()
        comm.blur(N, M, lin, lout)
        torch.cuda.synchronize()
        Rb, Db = oracle.blur(img, rows=np.arange(b0, b0 + brows))
        got = lout.cpu().numpy().astype(np.float64)
        out["blur_err"] = float(np.max(np.abs(got - Rb) / Db))
        out["blur_bytes"] = comm.bytes_received() - before
        out["blur_bytes_expected"] = 0 if rank == world - 1 else 2 * 3 * M * 4
        out["check"] = comm.check()
        comm.close()
    except Exception as e:  # reported to the parent, which fails the test
        out["error"] = repr(e)
    q.put((rank, out))
    dist.destroy_process_group()


def test_multi_rank_nccl_broadcast_and_allgather():
    import torch
    world = torch.cuda.device_count()
    if world < 2:
        pytest.skip(f"needs >= 2 GPUs for NCCL ranks (found {world})")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(world):
        o = res[r]
        assert "error" not in o, o
        assert o["bcast_err"] <= TOL and o["ag_err"] <= TOL, o
        assert o["bcast_B_equal"] and o["ag_B_equal"] and o["fused_B_equal"], o
        assert o["fused_err"] <= TOL, o
        assert o["bcast_bytes"] == o["bcast_bytes_expected"], o
        assert o["ag_bytes"] == o["ag_bytes_expected"], o
        assert o["blur_err"] <= 1e-6 and o["blur_bytes"] == o["blur_bytes_expected"], o
        assert o["summa_err"] <= TOL, o
        assert o["check"], o
