"""Host-side logic of the row-sharded multi-GPU mode, world_size 2 over gloo on
CPU: NCCL unique-id bootstrap through a torch.distributed group, the row
partition (every row owned exactly once, "distributed across the
nodes by rows"; no gather of C), and the K-chunk broadcast
schedule (chunks tile [0,k) once: message conservation, each non-root rank
receives exactly k*ldb*4 bytes)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # 1. unique-id bootstrap: rank 0 creates, everyone receives identical bytes
        obj = [tm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        out["ids_equal"] = all(i == ids[0] for i in ids) and len(ids[0]) == 128
        # 2. row partition agreed by all ranks, covering [0, m) once
        parts = {}
        for m in (0, 1, 7, 1060, 16384, 16387):
            mine = tm.dist_rows(m, world, rank)
            allp = [None] * world
            dist.all_gather_object(allp, mine)
            rows = []
            for r0, nr in allp:
                rows.extend(range(r0, r0 + nr))
            parts[m] = rows == list(range(m))
        out["partition_ok"] = all(parts.values())
        # 3. chunk schedule identical on all ranks and conserving bytes
        sched = {k: tm.dist_chunks(k, world) for k in (1, 33, 576, 1060, 16384)}
        alls = [None] * world
        dist.all_gather_object(alls, sched)
        out["schedule_same"] = all(s == alls[0] for s in alls)
        ok = True
        for k, ch in sched.items():
            pos = 0
            for k0, kr in ch:
                ok &= (k0 == pos) and kr > 0
                pos += kr
            ok &= pos == k
            ok &= all(k0 % 32 == 0 for k0, _ in ch)
        out["schedule_tiles_k"] = bool(ok)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_dist_host_logic_world2_gloo():
    try:
        import paper_1804_10694_b200 as tm
        tm.unique_id()
    except Exception as e:  # NCCL not loadable on this host
        pytest.skip(f"NCCL unavailable: {e}")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r] == {"ids_equal": True, "partition_ok": True, "schedule_same": True,
                          "schedule_tiles_k": True}, res[r]


def test_chunk_schedule_single_process():
    import paper_1804_10694_b200 as tm
    assert tm.dist_chunks(16384, 1) == [(0, 16384)]  # P == 1: no chunking (== tm_sgemm)
    # geometric chunks (dist.cpp chunk_plan): 512, 1024, 2048, 4096, then the
    # last absorbs a remainder of at most half its size
    assert tm.dist_chunks(16384, 8) == [(0, 512), (512, 1024), (1536, 2048), (3584, 4096), (7680, 8704)]
    assert tm.dist_chunks(1100, 2) == [(0, 512), (512, 588)]        # larger remainder: its own chunk
    assert tm.dist_chunks(4096, 4) == [(0, 512), (512, 1024), (1536, 2560)]
    assert tm.dist_chunks(600, 4) == [(0, 600)]                      # below two first chunks: one
    for k in (1, 31, 513, 1024, 5000, 65536, 1 << 20):
        ch = tm.dist_chunks(k, 3)
        assert ch[0][0] == 0 and sum(kr for _, kr in ch) == k and len(ch) <= 16
        assert all(a + ka == b for (a, ka), (b, _) in zip(ch, ch[1:]))
        assert all(k0 % 32 == 0 for k0, _ in ch)
        assert all(kb >= ka for (_, ka), (_, kb) in zip(ch, ch[1:-1]))  # non-decreasing before the last
    assert tm.dist_chunks(0, 4) == []


def _soak_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import time
    import torch
    import torch.distributed as dist
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        now = time.time()
        # rank 0's own clock says the soak is over, rank 1's says go on: both must go on
        mixed = bench.soak_more(torch, dist, world, now - 5.0 if rank == 0 else now)
        done = bench.soak_more(torch, dist, world, now - 5.0)  # every clock says over
        q.put((rank, mixed, done))
    finally:
        dist.destroy_process_group()


def test_bench_soak_decision_is_collective():
    """bench.py's N > 1 soak loop: every step is a collective, so the decision
    to keep soaking must be the same on every rank (a per-rank wall-clock test
    once left one rank in a broadcast the other never joined)."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_soak_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert [r[1] for r in res] == [True, True] and [r[2] for r in res] == [False, False], res
