"""Transposed operands (BLAS op()) and the column-major
BLAS entry, against the oracle's op(A), op(B) (pinned in test_oracle.py)."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
TOL = 1e-5
SIMT, TF32X3, AUTO = 2, 1, 0


def _pad(x):
    return (x + 3) // 4 * 4


def _stored(g, rows, cols, ld):
    buf = si.uniform(g, (rows, ld))
    return buf[:, :cols]


def _dev(x):
    import torch
    base = x.base if x.base is not None else x
    t = torch.from_numpy(np.ascontiguousarray(base)).cuda()
    return t[:x.shape[0], :x.shape[1]]


@pytest.mark.parametrize("algo", [SIMT, TF32X3])
@pytest.mark.parametrize("opa,opb", [("N", "T"), ("T", "N"), ("T", "T"), ("N", "N")])
@pytest.mark.parametrize("shape", [(300, 260, 200), (1060, 1060, 1060), (129, 33, 517), (5, 7, 3)])
def test_op_parity(algo, opa, opb, shape):
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = shape
    g = si.rng(m * 3 + n * 5 + k)
    ar, ac = (k, m) if opa == "T" else (m, k)
    br, bc = (n, k) if opb == "T" else (k, n)
    A = _stored(g, ar, ac, _pad(ac) + 4)
    B = _stored(g, br, bc, _pad(bc))
    C0 = _stored(g, m, n, _pad(n))
    dA, dB, dC = _dev(A), _dev(B), _dev(C0)
    tm.sgemm_op(dA, dB, dC, si.ALPHA, si.BETA, opa, opb, algo=algo)
    torch.cuda.synchronize()
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, opa=opa, opb=opb)
    assert float(np.max(oracle.normalized_error(dC.cpu().numpy(), R, D))) <= TOL


@pytest.mark.parametrize("opa,opb", [("N", "T"), ("T", "N"), ("T", "T")])
def test_op_tensor_core_configs_and_streamk(opa, opb):
    import os
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 777, 1000, 900
    g = si.rng(5)
    A = _stored(g, *((k, m) if opa == "T" else (m, k)), _pad(m if opa == "T" else k))
    B = _stored(g, *((n, k) if opb == "T" else (k, n)), _pad(k if opb == "T" else n))
    C0 = _stored(g, m, n, _pad(n))
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, opa=opa, opb=opb)
    for cfg in ["2,128,0", "2,128,1", "2,64,1", "2,32,0", "1,128,0", "1,64,1", "1,32,0"]:
        os.environ["TM_TC_CONFIG"] = cfg
        try:
            dA, dB, dC = _dev(A), _dev(B), _dev(C0)
            tm.sgemm_op(dA, dB, dC, si.ALPHA, si.BETA, opa, opb, algo=TF32X3)
            torch.cuda.synchronize()
        finally:
            del os.environ["TM_TC_CONFIG"]
        assert float(np.max(oracle.normalized_error(dC.cpu().numpy(), R, D))) <= TOL, cfg


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
def test_colmajor_blas_entry(ta, tb):
    """Column-major C = alpha op(A) op(B) + beta C (reference-BLAS sgemm
    argument convention), checked against the oracle on the same data."""
    import ctypes
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 300, 200, 150
    g = si.rng(9)
    # column-major matrices are the transposes of the row-major arrays we hold
    Acm = si.uniform(g, (k, m) if ta == "N" else (m, k))   # row-major view of column-major A
    Bcm = si.uniform(g, (n, k) if tb == "N" else (k, n))
    Ccm = si.uniform(g, (n, m))                              # row-major view of column-major C (m x n)
    A_cm_mat = Acm.T                         # the column-major matrix A as stored (rows x cols)
    B_cm_mat = Bcm.T
    opA = A_cm_mat if ta == "N" else A_cm_mat.T
    opB = B_cm_mat if tb == "N" else B_cm_mat.T
    C_cm_mat = Ccm.T
    R, D = oracle.sgemm(si.ALPHA, np.ascontiguousarray(opA), np.ascontiguousarray(opB), si.BETA,
                        np.ascontiguousarray(C_cm_mat))
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (Acm, Bcm, Ccm))
    lda, ldb, ldc = Acm.shape[1], Bcm.shape[1], Ccm.shape[1]
    st = tm.lib.tm_sgemm_colmajor(ta.encode(), tb.encode(), m, n, k, si.ALPHA, ctypes.c_void_p(dA.data_ptr()), lda,
                                  ctypes.c_void_p(dB.data_ptr()), ldb, si.BETA, ctypes.c_void_p(dC.data_ptr()), ldc,
                                  None)
    assert st == 0
    torch.cuda.synchronize()
    Cgpu = dC.cpu().numpy().T  # back to the m x n mathematical matrix
    assert float(np.max(oracle.normalized_error(Cgpu, R, D))) <= TOL


@pytest.mark.parametrize("opa,opb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("algo,tol", [(1, 1e-5), (4, 1e-5), (3, 2.0 ** -9 + 2.0 ** -14)])
def test_op_hybrid_streamk_every_precision(opa, opb, algo, tol):
    """The hybrid stream-K schedule (partial wave + one wave split, then whole
    tiles: 170 tiles of 256 x 128 on 74 clusters, 22 K-blocks) under every
    operand layout and precision variant (3xTF32, BF16x9 at 1e-5; 1xTF32 at its
    own bound, include/tm.h), against the oracle on sampled rows."""
    import os
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 2500, 2100, 700
    g = si.rng(11 + algo)
    A = _stored(g, *((k, m) if opa == "T" else (m, k)), _pad(m if opa == "T" else k))
    B = _stored(g, *((n, k) if opb == "T" else (k, n)), _pad(k if opb == "T" else n))
    C0 = _stored(g, m, n, _pad(n))
    os.environ["TM_TC_CONFIG"] = "2,64,1"
    try:
        dA, dB, dC = _dev(A), _dev(B), _dev(C0)
        tm.sgemm_op(dA, dB, dC, si.ALPHA, si.BETA, opa, opb, algo=algo)
        torch.cuda.synchronize()
    finally:
        del os.environ["TM_TC_CONFIG"]
    assert tm.streamk_region(10 * 17, 22, 74) == (22 + 74, 74)
    rows = si.sample_rows(m, count=96)
    Ar = A[rows] if opa == "N" else A[:, rows]
    R, D = oracle.sgemm(si.ALPHA, np.ascontiguousarray(Ar), np.ascontiguousarray(B), si.BETA,
                        np.ascontiguousarray(C0[rows]), opa=opa, opb=opb)
    err = float(np.max(oracle.normalized_error(dC.cpu().numpy()[rows], R, D)))
    assert err <= tol, (opa, opb, algo, err)
