"""CUDA-graph capture of the GEMM (streams and graphs instead of a tracing
compiler): tm_sgemm enqueues only kernels, memsets and (under capture) a
graph-owned workspace allocation, so a captured call replays correctly --
including stream-K schedules, whose epoch flags are cleared inside the graph
before each replay (csrc/api.cpp streamk_workspace)."""
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("cfg", [None, "2,64,1", "1,128,1", "2,128,0"])
def test_captured_sgemm_replays(cfg):
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 1060, 1060, 1060
    A, B, _ = si.matrices(m, n, k, 41)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros((m, n), dtype=torch.float32, device="cuda")
    if cfg:
        os.environ["TM_TC_CONFIG"] = cfg
    try:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            tm.sgemm_ex(dA, dB, dC, si.ALPHA, si.BETA, tm.ALGO_TF32X3)  # warm-up: sizes the workspace
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            tm.sgemm_ex(dA, dB, dC, si.ALPHA, si.BETA, tm.ALGO_TF32X3)
    finally:
        if cfg:
            del os.environ["TM_TC_CONFIG"]
    for rep in range(3):
        # new A every replay: stale stream-K partials from the previous replay
        # would then give a wrong result (they depend on A and B, not on C0)
        A = si.uniform(si.rng(200 + rep), (m, k))
        C0 = si.uniform(si.rng(100 + rep), (m, n))
        dA.copy_(torch.from_numpy(A))
        dC.copy_(torch.from_numpy(C0))
        g.replay()
        torch.cuda.synchronize()
        R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
        err = float(np.max(oracle.normalized_error(dC.cpu().numpy(), R, D)))
        assert err <= TOL, (cfg, rep, err)


@pytest.mark.parametrize("cfg", ["2,64,1", "2,128,0", "2,128,1"])
def test_default_graph_idiom_and_replay_on_other_streams(cfg):
    """The standard torch.cuda.graph idiom (warm-up on a side stream, capture on
    torch's own capture stream, no stream argument): stream-K and wave-barrier
    launches allocate their workspace inside the graph, so capture needs no
    prior call on the capturing stream, and replays on other streams, two graphs
    of the same shape, and direct calls in between do not share flags."""
    import torch
    import paper_1804_10694_b200 as tm
    # 2,128,0 at 4096 x 4096 x 2048: 256 tiles on 74 clusters, 64 K-blocks -> wave barrier;
    # 2,128,1 there: hybrid stream-K (34 tiles split) + the barrier over its 3 whole waves,
    # whose counter is slot 0 of the graph-owned stream-K flags
    m, n, k = (1060, 1060, 1060) if cfg == "2,64,1" else (4096, 4096, 2048)
    A, B, _ = si.matrices(m, n, k, 43)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC1 = torch.zeros((m, n), device="cuda")
    dC2 = torch.zeros((m, n), device="cuda")
    os.environ["TM_TC_CONFIG"] = cfg
    try:
        graphs = []
        for dC in (dC1, dC2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                tm.sgemm_ex(dA, dB, dC, si.ALPHA, si.BETA, tm.ALGO_TF32X3)
            graphs.append(g)
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        for rep in range(2):
            C0 = si.uniform(si.rng(300 + rep), (m, n))
            dC1.copy_(torch.from_numpy(C0))
            dC2.copy_(torch.from_numpy(C0))
            torch.cuda.synchronize()
            for g, s in zip(graphs, streams):
                with torch.cuda.stream(s):
                    g.replay()
            dD = torch.from_numpy(C0).cuda()
            tm.sgemm_ex(dA, dB, dD, si.ALPHA, si.BETA, tm.ALGO_TF32X3)  # direct call while graphs run
            torch.cuda.synchronize()
            rows = si.sample_rows(m, count=64)
            R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, rows=rows)
            for out in (dC1, dC2, dD):
                err = float(np.max(oracle.normalized_error(out.cpu().numpy()[rows], R, D)))
                assert err <= TOL, (cfg, rep, err)
            assert torch.equal(dC1, dC2) and torch.equal(dC1, dD)  # deterministic across paths
    finally:
        del os.environ["TM_TC_CONFIG"]
