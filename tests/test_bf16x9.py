"""BF16x9 precision variant (TM_ALGO_BF16X9, the
precision generalisation of the paper's auto-tuned sgemm variants, PAPER.md:
831-832): each fp32 operand split in the kernel into three bf16 pieces that
represent it exactly, all nine products on kind::f16 tcgen05 MMAs, the 3xTF32
path's accumulation (include/tm.h).  Against the fp64 oracle at the north_star
1e-5 on the same seeded inputs, every layout and compiled tile configuration,
ragged shapes, stream-K, deep K with all-positive inputs (the accumulation
stress case), integer inputs bit-exact, and an error case that separates it
from 3xTF32 (products of full-mantissa values: exact here, 2^-19 there)."""
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
BF16X9, TF32X3 = 4, 1
TOL = 1e-5


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _run(A, B, C0, alpha, beta, opa="N", opb="N", algo=BF16X9, config=None):
    import torch
    import paper_1804_10694_b200 as tm
    dA, dB, dC = _dev(A), _dev(B), _dev(C0)
    if config:
        os.environ["TM_TC_CONFIG"] = config
    try:
        tm.sgemm_op(dA, dB, dC, alpha, beta, opa, opb, algo=algo)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("TM_TC_CONFIG", None)
    return dC.cpu().numpy()


def _operands(g, m, n, k, opa, opb, gen=si.uniform):
    A = gen(g, (k, m) if opa == "T" else (m, k))
    B = gen(g, (n, k) if opb == "T" else (k, n))
    return A, B, gen(g, (m, n))


def test_plan_name():
    import paper_1804_10694_b200 as tm
    assert tm.plan_name(1024, 1024, 1024, A_ptr=1 << 12, B_ptr=1 << 24, C_ptr=1 << 30, algo=BF16X9) == "bf16x9"


@pytest.mark.parametrize("opa,opb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("config", ["2,128,0", "2,64,1", "1,128,1", "1,64,0"])
def test_bf16x9_parity_layouts_and_configs(opa, opb, config):
    m, n, k = 300, 260, 516   # partial M/N tiles, K tail of 4
    g = si.rng(sum(map(ord, opa + opb + config)))
    A, B, C0 = _operands(g, m, n, k, opa, opb)
    C = _run(A, B, C0, si.ALPHA, si.BETA, opa, opb, config=config)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, opa=opa, opb=opb)
    assert float(np.max(oracle.normalized_error(C, R, D))) <= TOL


@pytest.mark.parametrize("shape", [(1060, 1060, 1060), (129, 68, 36), (4096, 256, 4096), (2048, 2048, 8192)])
def test_bf16x9_shapes_and_deep_k(shape):
    m, n, k = shape
    g = si.rng(m + n + k)
    for gen in (si.uniform, lambda g, s: si.uniform(g, s, 0.0, 1.0)):  # zero-mean and all-positive
        A, B, C0 = _operands(g, m, n, k, "N", "N", gen)
        C = _run(A, B, C0, si.ALPHA, si.BETA)
        rows = si.sample_rows(m, count=96)
        R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, rows=rows)
        assert float(np.max(oracle.normalized_error(C[rows], R, D))) <= TOL, shape


def test_bf16x9_integer_inputs_bit_exact_and_beta_zero():
    m, n, k = 900, 700, 1500
    A, B, C0 = si.matrices(m, n, k, 14, kind="integer")
    C = _run(A, B, C0, 1.5, 0.5, config="2,128,1")
    R, _ = oracle.sgemm(1.5, A, B, 0.5, C0)
    assert np.array_equal(C.astype(np.float64), R)
    A, B, C0 = si.matrices(300, 260, 200, 15)
    C = _run(A, B, np.full_like(C0, np.nan), 2.0, 0.0)  # beta = 0: C is not read
    R, D = oracle.sgemm(2.0, A, B, 0.0, None)
    assert np.all(np.isfinite(C)) and float(np.max(oracle.normalized_error(C, R, D))) <= TOL


def test_bf16x9_products_exact_where_3xtf32_is_not():
    """k = 8: a handful of products of full-mantissa values, so the result is
    dominated by representation error.  BF16x9 represents every operand exactly
    (its error is the fp32 accumulation only, a few 2^-24); 3xTF32 truncates hi
    and drops lo*lo (bound 2^-19 per product)."""
    m, n, k = 512, 512, 8
    g = si.rng(16)
    A, B, C0 = _operands(g, m, n, k, "N", "N", lambda g, s: si.uniform(g, s, 1.0, 2.0))
    R, D = oracle.sgemm(1.0, A, B, 0.0, None)
    e9 = float(np.max(oracle.normalized_error(_run(A, B, C0, 1.0, 0.0, config="2,128,0"), R, D)))
    e3 = float(np.max(oracle.normalized_error(_run(A, B, C0, 1.0, 0.0, algo=TF32X3, config="2,128,0"), R, D)))
    assert e9 <= 2.0 ** -21, e9
    assert e9 < e3, (e9, e3)
