"""CUDA-graph capture of the GEMM (streams and graphs instead of a tracing
compiler): tm_sgemm enqueues only kernels and memsets, so a call captured once
(after one warm-up call that sizes the library's stream-K workspace) replays
correctly -- including stream-K schedules, whose per-launch epoch flags are
cleared inside the graph before each replay (csrc/api.cpp streamk_workspace)."""
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


def test_capture_without_workspace_is_an_error_not_a_hang():
    """A stream-K launch whose workspace does not exist yet cannot allocate it
    during capture: the call reports TM_ERR_INVALID_VALUE instead."""
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 1060, 1060, 1060
    dA = torch.zeros((m, k), device="cuda")
    dB = torch.zeros((k, n), device="cuda")
    dC = torch.zeros((m, n), device="cuda")
    s = torch.cuda.Stream()  # fresh stream: no workspace yet
    os.environ["TM_TC_CONFIG"] = "2,64,1"
    g = torch.cuda.CUDAGraph()
    try:
        with pytest.raises(tm.TmError):
            with torch.cuda.graph(g, stream=s):
                tm.sgemm_ex(dA, dB, dC, 1.0, 0.5, tm.ALGO_TF32X3)
    finally:
        del os.environ["TM_TC_CONFIG"]
    torch.cuda.synchronize()
