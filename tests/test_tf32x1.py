"""1xTF32 precision variant (TM_ALGO_TF32X1): one
tcgen05 kind::tf32 MMA per K step on the raw operands, which the tensor core
truncates to TF32.  Bound (include/tm.h): per product |a_hi b_hi - ab| <=
2^-9 |a||b|, plus the 3xTF32 path's accumulation bound -> max normalized error
<= 2^-9 + 2^-14 for k <= 4096.  Checked against the fp64 oracle on the same
seeded inputs, every layout; integer inputs (exact in TF32) are bit-exact."""
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
TF32X1 = 3
TOL1 = 2.0 ** -9 + 2.0 ** -14


def _pad(x):
    return (x + 3) // 4 * 4


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _run(A, B, C0, alpha, beta, opa, opb):
    import torch
    import paper_1804_10694_b200 as tm
    dA, dB, dC = _dev(A), _dev(B), _dev(C0)
    tm.sgemm_op(dA, dB, dC, alpha, beta, opa, opb, algo=TF32X1)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


def _operands(g, m, n, k, opa, opb, gen):
    A = gen(g, (k, m) if opa == "T" else (m, k))
    B = gen(g, (n, k) if opb == "T" else (k, n))
    C0 = gen(g, (m, n))
    return A, B, C0


@pytest.mark.parametrize("opa,opb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("shape", [(300, 260, 200), (1060, 1060, 1060), (132, 36, 516), (4096, 256, 4096)])  # ld = dim: 4-aligned
def test_tf32x1_parity(opa, opb, shape):
    m, n, k = shape
    g = si.rng(m + 7 * n + 13 * k)
    A, B, C0 = _operands(g, m, n, k, opa, opb, si.uniform)
    C = _run(A, B, C0, si.ALPHA, si.BETA, opa, opb)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, opa=opa, opb=opb)
    e = float(np.max(oracle.normalized_error(C, R, D)))
    assert e <= TOL1, e
    assert e > 1e-6, e  # really one TF32 pass (3xTF32 / fp32 would be ~1e-7)


@pytest.mark.parametrize("opa,opb", [("N", "N"), ("T", "T")])
def test_tf32x1_integer_inputs_bit_exact(opa, opb):
    """Integers in [-4, 4] are exact in TF32 (no truncation) and every partial
    sum is an exactly representable fp32 integer: the result equals the oracle."""
    m, n, k = 260, 300, 700
    g = si.rng(31)
    gen = lambda g, shape: si.integers(g, shape)  # noqa: E731
    A, B, C0 = _operands(g, m, n, k, opa, opb, gen)
    C = _run(A, B, C0, si.ALPHA, si.BETA, opa, opb)
    R, _ = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, opa=opa, opb=opb)
    assert np.array_equal(C.astype(np.float64), R)


@pytest.mark.parametrize("cfg", ["2,128,0", "2,128,1", "2,64,1", "2,32,0", "1,128,1", "1,64,0", "1,32,1"])
def test_tf32x1_configs(cfg):
    m, n, k = 777, 1000, 900
    A, B, C0 = si.matrices(m, n, k, 5)
    os.environ["TM_TC_CONFIG"] = cfg
    try:
        C = _run(A, B, C0, si.ALPHA, si.BETA, "N", "N")
    finally:
        del os.environ["TM_TC_CONFIG"]
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    assert float(np.max(oracle.normalized_error(C, R, D))) <= TOL1, cfg


def test_tf32x1_beta_zero_does_not_read_C():
    m, n, k = 200, 136, 96
    A, B, C0 = si.matrices(m, n, k, 8)
    C0[:] = np.nan
    C = _run(A, B, C0, 1.0, 0.0, "N", "N")
    R, D = oracle.sgemm(1.0, A, B, 0.0, C0)
    assert np.all(np.isfinite(C))
    assert float(np.max(oracle.normalized_error(C, R, D))) <= TOL1
