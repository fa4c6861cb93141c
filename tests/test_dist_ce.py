"""Copy-engine chain broadcast (tm_ce_*, tm_sgemm_dist_ce; SURVEY.md 8(f)
item 3) with real processes: `world` ranks that all share the single GPU of
the box (CUDA IPC works between processes on one device), bootstrapped over
gloo.  Each rank's C shard must match the oracle at the north_star 1e-5
(rows distributed; no gather); every non-root
B ends equal to the root's; each non-root receives exactly k*ldb*4 bytes per
call; repeated calls exercise the per-call credits and epochs (root != 0,
uneven rows, chunked and fused schedules)."""
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
    torch.cuda.set_device(0)  # every rank on the one GPU
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        cc = tm.CeComm(rank, world)
        m, n, k, root = 1061, 300, 1100, world - 1
        A, B, C0 = si.matrices(m, n, k, seed=66)
        r0, rows = tm.dist_rows(m, world, rank)
        R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, rows=np.arange(r0, r0 + rows))
        dA = torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda()
        dB = torch.from_numpy(B).cuda() if rank == root else torch.full((k, n), float("nan"), device="cuda")
        handles = cc.exchange(dB)
        errs, equal = [], []
        for it, fused in enumerate((False, True, False, True)):
            if rank != root:
                dB.fill_(float("nan"))
            dC = torch.from_numpy(np.ascontiguousarray(C0[r0:r0 + rows])).cuda()
            cc.sgemm(m, n, k, dA, dB, dC, si.ALPHA, si.BETA, root=root, fused=fused, handles=handles)
            torch.cuda.synchronize()
            errs.append(float(np.max(oracle.normalized_error(dC.cpu().numpy(), R, D))) if rows else 0.0)
            equal.append(bool(np.array_equal(dB.cpu().numpy(), B)))
            dist.barrier()  # the next call's NaN refill must not race a slower peer's push
        out["errs"] = errs
        out["B_equal"] = equal
        out["bytes"] = cc.bytes_received()
        out["bytes_expected"] = 0 if rank == root else 4 * k * n * 4
        cc.close()
    except Exception as e:  # reported to the parent, which fails the test
        out["error"] = repr(e)
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ce_chain_processes_sharing_one_gpu(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=300) for _ in procs)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    for r in range(world):
        o = res[r]
        assert "error" not in o, o
        assert max(o["errs"]) <= TOL, o
        assert all(o["B_equal"]), o
        assert o["bytes"] == o["bytes_expected"], o
