"""The latency-bound small-GEMM kernel (csrc/small_gemm.cu), which AUTO uses
for m*n*k <= 2^22 and k <= 256 (BASELINE.json configs[0] = C1, 64^3), against the oracle:
ragged shapes around its 32/64 tiles and 32-deep K slices, every op() layout,
padded leading dimensions with guard bands, beta = 0 with NaN in C, integer
inputs bit-exact (fp32 FMA chains of exact products)."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si
from gpu_util import SENTINEL, max_err, run

pytestmark = pytest.mark.gpu
TOL = 1e-5
AUTO = 0


def test_c1_takes_the_small_kernel():
    import paper_1804_10694_b200 as tm
    assert tm.plan_name(64, 64, 64, si.ALPHA, si.BETA, 1 << 12, 64, 1 << 16, 64, 1 << 24, 64) == "simt_small"


@pytest.mark.parametrize("shape", [(64, 64, 64), (1, 1, 1), (33, 31, 65), (64, 64, 1), (5, 200, 7), (200, 3, 256),
                                   (97, 129, 33), (128, 128, 256), (600, 500, 12), (1000, 16, 255)])
def test_small_parity_and_guard_band(shape):
    import paper_1804_10694_b200 as tm
    m, n, k = shape
    assert tm.plan_name(m, n, k, si.ALPHA, si.BETA, 1 << 12, k + 3, 1 << 16, n + 5, 1 << 30, n + 2) == "simt_small"
    A, B, C0 = si.matrices(m, n, k, seed=sum(shape), lda=k + 3, ldb=n + 5, ldc=n + 2)
    C, buf = run(A, B, C0, si.ALPHA, si.BETA, AUTO, lda=k + 3, ldb=n + 5, ldc=n + 2, guard_rows=2)
    assert max_err(C, A, B, C0, si.ALPHA, si.BETA) <= TOL
    assert np.all(buf[:m, n:] == SENTINEL) and np.all(buf[m:] == SENTINEL)  # nothing outside m x n written


@pytest.mark.parametrize("opa,opb", [("N", "T"), ("T", "N"), ("T", "T")])
def test_small_transposes(opa, opb):
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 70, 90, 110
    A, B, C0 = si.matrices(m, n, k, seed=5)
    At = np.ascontiguousarray(A.T) if opa == "T" else A
    Bt = np.ascontiguousarray(B.T) if opb == "T" else B
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (At, Bt, C0))
    tm.sgemm_op(dA, dB, dC, si.ALPHA, si.BETA, opa, opb)
    torch.cuda.synchronize()
    R, D = oracle.sgemm(si.ALPHA, At, Bt, si.BETA, C0, opa=opa, opb=opb)
    assert float(np.max(oracle.normalized_error(dC.cpu().numpy(), R, D))) <= TOL


def test_small_beta_zero_nan_c_and_integer_bit_exact():
    m, n, k = 100, 120, 140
    A, B, C0 = si.matrices(m, n, k, seed=9)
    C, _ = run(A, B, C0, si.ALPHA, 0.0, AUTO, c_fill=np.nan)
    assert np.all(np.isfinite(C)) and max_err(C, A, B, C0, si.ALPHA, 0.0) <= TOL
    A, B, C0 = si.matrices(m, n, k, seed=10, kind="integer")
    C, _ = run(A, B, C0, 1.5, 0.5, AUTO)
    R, _ = oracle.sgemm(1.5, A, B, 0.5, C0)
    assert np.array_equal(C.astype(np.float64), R)
