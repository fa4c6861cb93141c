"""Measured configuration choice (tm_sgemm_tune; the
paper auto-tuned its sgemm's tile sizes): the host-side
cache (CPU) and tuning on the device (GPU)."""
import ctypes
import os

import numpy as np
import pytest

import paper_1804_10694_b200 as tm

TC = 3  # plan_config path code: tensor cores


@pytest.fixture(autouse=True)
def _clean_cache():
    tm.tune_cache_clear()
    yield
    tm.tune_cache_clear()


def test_cache_file_roundtrip_and_planner_use(tmp_path):
    default = tm.plan_config(1060, 1060, 1060, beta=0.5)
    default_b0 = tm.plan_config(1060, 1060, 1060, beta=0.0)
    other = tm.plan_config(1061, 1060, 1060, beta=0.5)
    assert default[0] == TC
    f = tmp_path / "tune.txt"
    f.write_text("# comment\n"
                 "1060 1060 1060 0 0 1 148 1 32 0\n"      # valid: beta != 0, NN
                 "1060 1060 1060 0 0 1 148 3 32 0\n"      # cg 3: invalid
                 "1060 1060 1060 0 0 1 148 1 48 0\n"      # bn 48: invalid
                 "-5 1060 1060 0 0 1 148 1 32 0\n"        # negative m
                 "not a line\n"
                 "777 1000 900 1 0 1 148 2 128 1\n")      # valid: A transposed
    assert tm.tune_cache_load(str(f)) == 2
    assert tm.tune_cache_size() == 2
    # the planner uses the cached entry for exactly that key ...
    assert tm.plan_config(1060, 1060, 1060, beta=0.5) == (TC, 1, 32, 0)
    # ... not for beta == 0, another shape, or another layout
    assert tm.plan_config(1060, 1060, 1060, beta=0.0) == default_b0
    assert tm.plan_config(1061, 1060, 1060, beta=0.5) == other
    assert tm.plan_config(777, 1000, 900, beta=0.5, opa="T", lda=780) == (TC, 2, 128, 1)
    # TF32X1 and SIMT never take tuned tensor-core entries
    assert tm.plan_config(1060, 1060, 1060, beta=0.5, algo=tm.ALGO_SIMT_F32)[0] == 4
    # save -> clear -> load reproduces the cache
    g = tmp_path / "saved.txt"
    tm.tune_cache_save(str(g))
    tm.tune_cache_clear()
    assert tm.tune_cache_size() == 0
    assert tm.plan_config(1060, 1060, 1060, beta=0.5) == default
    assert tm.tune_cache_load(str(g)) == 2
    assert tm.plan_config(1060, 1060, 1060, beta=0.5) == (TC, 1, 32, 0)
    with pytest.raises(OSError):
        tm.tune_cache_load(str(tmp_path / "missing.txt"))


def test_tune_rejects_bad_arguments_on_host():
    L = tm.lib
    vp = ctypes.c_void_p
    args = lambda **kw: dict(dict(opa=0, opb=0, m=64, n=64, k=64, alpha=1.0, A=1 << 12, lda=64, B=1 << 16, ldb=64,
                                  beta=0.0, C=1 << 24, ldc=64, reps=3), **kw)

    def call(**kw):
        a = args(**kw)
        return L.tm_sgemm_tune(a["opa"], a["opb"], a["m"], a["n"], a["k"], a["alpha"], vp(a["A"]), a["lda"],
                               vp(a["B"]), a["ldb"], a["beta"], vp(a["C"]), a["ldc"], None, a["reps"], None, None,
                               None, None)
    assert call(reps=0) == 1
    assert call(alpha=0.0) == 1
    assert call(k=0) == 1
    assert call(opa=2) == 1
    assert call(lda=63) == 1                 # lda < k
    assert call(A=(1 << 12) + 4) == 1        # misaligned: no tensor-core plan
    assert call(C=1 << 12) == 1              # C overlaps A


@pytest.mark.gpu
@pytest.mark.parametrize("opa,opb,beta", [("N", "N", 0.5), ("T", "N", 0.0), ("N", "T", 0.5)])
def test_tune_on_device_keeps_c_and_results_correct(opa, opb, beta):
    import torch
    import oracle
    import seeded_inputs as si
    m, n, k = 1060, 1060, 1060
    g = si.rng(77)
    A = si.uniform(g, (k, m) if opa == "T" else (m, k))
    B = si.uniform(g, (n, k) if opb == "T" else (k, n))
    C0 = si.uniform(g, (m, n))
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, B, C0))
    cg, bn, sk, ms = tm.tune(dA, dB, dC, si.ALPHA, beta, opa, opb, reps=3)
    torch.cuda.synchronize()
    assert cg in (1, 2) and bn in (32, 64, 128) and sk in (0, 1) and ms > 0
    assert np.array_equal(dC.cpu().numpy(), C0)          # tuning never writes the caller's C
    assert tm.tune_cache_size() == 1
    cfg = tm.plan_config(m, n, k, si.ALPHA, beta, dA.data_ptr(), dA.stride(0), dB.data_ptr(), dB.stride(0),
                         dC.data_ptr(), dC.stride(0), opa, opb)
    assert cfg == (TC, cg, bn, sk)
    tm.sgemm_op(dA, dB, dC, si.ALPHA, beta, opa, opb)
    torch.cuda.synchronize()
    R, D = oracle.sgemm(si.ALPHA, A, B, beta, C0, opa=opa, opb=opb)
    assert float(np.max(oracle.normalized_error(dC.cpu().numpy(), R, D))) <= 1e-5
