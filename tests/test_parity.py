"""GPU parity: every CUDA path against the CPU oracle on identical seeded inputs.

Bar (BASELINE.json north_star): max |C - R| / (|alpha| sum|A||B| + |beta||C0|)
<= 1e-5 per element, R and the denominator from oracle/ (fp64).  Integer-valued
inputs must be bit-exact on every path.
"""
import numpy as np
import pytest

import oracle
import seeded_inputs as si
from gpu_util import SENTINEL, max_err, run, to_dev

TOL = 1e-5
TC_CONFIGS = ["2,128", "2,64", "2,32", "1,128", "1,64", "1,32"]
SIMT, TF32X3, TF32X1, AUTO = 2, 1, 3, 0

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    torch.cuda.init()
    yield


@pytest.mark.parametrize("algo,config", [(SIMT, None)] + [(TF32X3, c) for c in TC_CONFIGS])
def test_c1_64(algo, config):
    m, n, k = si.CONFIGS["C1"]
    A, B, C0 = si.matrices(m, n, k, si.SEEDS["C1"])
    C, _ = run(A, B, C0, si.ALPHA, si.BETA, algo, config=config)
    assert max_err(C, A, B, C0, si.ALPHA, si.BETA) <= TOL


@pytest.mark.parametrize("algo,config", [(SIMT, None), (TF32X3, None)] + [(TF32X3, c) for c in TC_CONFIGS])
def test_c2_1060_partial_tiles(algo, config):
    m, n, k = si.CONFIGS["C2"]
    A, B, C0 = si.matrices(m, n, k, si.SEEDS["C2"])
    C, _ = run(A, B, C0, si.ALPHA, si.BETA, algo, config=config)
    assert max_err(C, A, B, C0, si.ALPHA, si.BETA) <= TOL


def test_tf32x1_data_movement():
    """Single-pass TF32 validates TMA/descriptor/epilogue data movement at a
    loose bound: per product |err| <= 2*2^-10 |a||b| (operand truncation)."""
    m, n, k = 300, 260, 200
    A, B, C0 = si.matrices(m, n, k, 77)
    C, _ = run(A, B, C0, 1.0, 0.0, TF32X1)
    e = max_err(C, A, B, C0, 1.0, 0.0)
    assert e <= 2.5 * 2.0 ** -10, e
    assert e > 1e-6  # it really is single-pass TF32 (not fp32)


RAGGED = [1, 2, 3, 5, 8, 9, 15, 16, 17, 31, 32, 33, 127, 128, 129, 255, 256, 257]


@pytest.mark.parametrize("algo", [SIMT, TF32X3])
def test_ragged_shapes(algo):
    g = si.rng(123)
    shapes = [(m, n, k) for m in (1, 17, 129, 257) for n in (1, 9, 33, 255) for k in (1, 8, 31, 257)]
    shapes += [tuple(int(x) for x in g.choice(RAGGED, 3)) for _ in range(20)]
    for (m, n, k) in shapes:
        # TF32X3 needs ld % 4 == 0: pad leading dimensions
        pad = lambda x: (x + 3) // 4 * 4
        lda, ldb, ldc = (pad(k), pad(n), pad(n)) if algo == TF32X3 else (k, n, n)
        A, B, C0 = si.matrices(m, n, k, seed=m * 10007 + n * 101 + k, lda=lda, ldb=ldb, ldc=ldc)
        C, _ = run(A, B, C0, si.ALPHA, si.BETA, algo, lda=lda, ldb=ldb, ldc=ldc)
        e = max_err(C, A, B, C0, si.ALPHA, si.BETA)
        assert e <= TOL, (m, n, k, e)


@pytest.mark.parametrize("algo,config", [(SIMT, None), (TF32X3, "2,128"), (TF32X3, "1,64"), (TF32X3, "2,32")])
def test_guard_band_untouched(algo, config):
    """Partial-tile separation: nothing outside m x n of C
    changes -- padding columns (ldc > n) and the rows after C keep a sentinel."""
    m, n, k = 300, 70, 45
    ldc = 80
    A, B, C0 = si.matrices(m, n, k, 5, lda=48, ldb=72)
    C, buf = run(A, B, C0, si.ALPHA, si.BETA, algo, lda=48, ldb=72, ldc=ldc, guard_rows=9, config=config)
    assert np.all(buf[:m, n:] == SENTINEL)
    assert np.all(buf[m:, :] == SENTINEL)
    assert max_err(C, A, B, C0, si.ALPHA, si.BETA) <= TOL


@pytest.mark.parametrize("algo", [SIMT, TF32X3])
def test_beta_zero_does_not_read_C(algo):
    m, n, k = 200, 136, 96
    A, B, _ = si.matrices(m, n, k, 6)
    Cnan = np.full((m, n), np.nan, dtype=np.float32)
    C, _ = run(A, B, Cnan, 1.5, 0.0, algo)
    assert np.all(np.isfinite(C))
    assert max_err(C, A, B, Cnan, 1.5, 0.0) <= TOL


@pytest.mark.parametrize("algo", [AUTO, SIMT, TF32X3])
def test_alpha_zero_and_k_zero(algo):
    m, n, k = 130, 68, 40
    g = si.rng(8)
    C0 = si.uniform(g, (m, n))
    Anan = np.full((m, k), np.nan, dtype=np.float32)
    Bnan = np.full((k, n), np.nan, dtype=np.float32)
    C, _ = run(Anan, Bnan, C0, 0.0, 0.5, algo)
    R, _ = oracle.sgemm(0.0, None, None, 0.5, C0, m=m, n=n, k=k)
    assert np.array_equal(C.astype(np.float64), R)  # beta*c is exact for beta = 0.5
    C, _ = run(Anan, Bnan, C0, 0.0, 0.0, algo, c_fill=np.nan)
    assert np.all(C == 0.0)
    C, _ = run(np.zeros((m, 0), np.float32), np.zeros((0, n), np.float32), C0, 1.5, 0.5, algo)
    assert np.array_equal(C.astype(np.float64), R)


@pytest.mark.parametrize("algo,config", [(SIMT, None)] + [(TF32X3, c) for c in TC_CONFIGS])
def test_integer_inputs_bit_exact(algo, config):
    """Integers in {-4..4} are exact in TF32 (hi = x, lo = 0) and every partial
    sum stays below 2^24, so every path must equal the oracle bit for bit."""
    m, n, k = 260, 200, 520
    A, B, C0 = si.matrices(m, n, k, 9, kind="integer")
    C, _ = run(A, B, C0, 1.5, 0.5, algo, config=config)
    R, _ = oracle.sgemm(1.5, A, B, 0.5, C0)
    assert np.array_equal(C.astype(np.float64), R)


@pytest.mark.parametrize("algo", [SIMT, TF32X3])
def test_deterministic(algo):
    m, n, k = 700, 520, 900
    A, B, C0 = si.matrices(m, n, k, 10)
    C1, _ = run(A, B, C0, si.ALPHA, si.BETA, algo)
    C2, _ = run(A, B, C0, si.ALPHA, si.BETA, algo)
    assert np.array_equal(C1, C2)


def test_identity_closed_form_tf32x3():
    """A = I: C = alpha*B + beta*C0 exactly up to the 3xTF32 representation
    error of B (lo truncation, <= 2^-19 relative) and the epilogue rounding."""
    n = 256
    g = si.rng(14)
    B = si.uniform(g, (n, 192))
    C0 = si.uniform(g, (n, 192))
    eye = np.eye(n, dtype=np.float32)
    C, _ = run(eye, B, C0, 1.5, 0.5, TF32X3)
    assert max_err(C, eye, B, C0, 1.5, 0.5) <= 2.0 ** -19 + 2.0 ** -23


@pytest.mark.parametrize("algo", [SIMT, TF32X3])
def test_c3_4096_sampled_rows(algo):
    m, n, k = si.CONFIGS["C3"]
    A, B, C0 = si.matrices(m, n, k, si.SEEDS["C3"])
    C, _ = run(A, B, C0, si.ALPHA, si.BETA, algo)
    rows = si.sample_rows(m, count=192)
    assert max_err(C, A, B, C0, si.ALPHA, si.BETA, rows=rows) <= TOL


@pytest.mark.parametrize("beta", [si.BETA, 0.0])
def test_c4_conv_im2col_sampled_rows(beta):
    A, B, C0 = si.im2col_conv()
    C, _ = run(A, B, C0, si.ALPHA, beta, AUTO)
    rows = si.sample_rows(A.shape[0], count=512)
    assert max_err(C, A, B, C0, si.ALPHA, beta, rows=rows) <= TOL


def test_c3b_8192_sampled_rows():
    m, n, k = si.CONFIGS["C3b"]
    A, B, C0 = si.matrices(m, n, k, si.SEEDS["C3b"])
    C, _ = run(A, B, C0, si.ALPHA, si.BETA, AUTO)
    rows = si.sample_rows(m, count=2 * m // 128 + 64, tile=128)  # both edge rows of every 128-row band
    assert len(rows) >= 2 * m // 128
    assert max_err(C, A, B, C0, si.ALPHA, si.BETA, rows=rows) <= TOL


@pytest.mark.parametrize("cfg,kind", [("C3b", "positive"), ("C5", "uniform"), ("C5", "positive")])
def test_large_k_accuracy_sampled_rows(cfg, kind):
    """Full-size configs (BASELINE.json configs[4] = C5, the bench workload)
    in the launch configuration bench.py times (AUTO path).  All-positive
    inputs stress the tensor core's round-toward-zero accumulation; K_c
    promotion keeps them inside the bar too."""
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = si.CONFIGS[cfg]
    A, B, C0 = si.matrices(m, n, k, si.SEEDS[cfg], kind=kind)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C0))
    tm.sgemm(dA, dB, dC, si.ALPHA, si.BETA)
    torch.cuda.synchronize()
    # both edge rows of every 128-row band (each CTA's rows of every 256x256
    # cluster tile) plus 64 seeded random rows -- SURVEY.md 8(d) "every tile row-band"
    rows = si.sample_rows(m, count=2 * m // 128 + 64, tile=128)
    assert len(rows) >= 2 * m // 128
    C = dC[torch.from_numpy(rows).cuda()].cpu().numpy()
    del dA, dB, dC
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, rows=rows)
    assert float(np.max(oracle.normalized_error(C, R, D))) <= TOL


@pytest.mark.parametrize("config", ["2,128,1", "2,64,1", "2,32,1", "1,128,1", "1,64,1", "1,32,1"])
@pytest.mark.parametrize("shape", [(1060, 1060, 1060), (300, 260, 5000), (777, 1000, 3000), (129, 65, 64),
                                   (2500, 2100, 700), (4100, 1000, 1200)])
def test_streamk_fixed_order_reduction(config, shape):
    """Stream-K (tiles split across clusters, partials reduced in cluster
    order through the workspace): parity and run-to-run bit-determinism.  The
    last two shapes have more tiles than clusters, so the hybrid schedule runs
    (the partial wave's tiles stream-K first, then whole tiles)."""
    m, n, k = shape
    pad = lambda x: (x + 3) // 4 * 4
    lda, ldb, ldc = pad(k), pad(n), pad(n)
    A, B, C0 = si.matrices(m, n, k, seed=m + n + k, lda=lda, ldb=ldb, ldc=ldc)
    C1, _ = run(A, B, C0, si.ALPHA, si.BETA, TF32X3, lda=lda, ldb=ldb, ldc=ldc, config=config)
    C2, _ = run(A, B, C0, si.ALPHA, si.BETA, TF32X3, lda=lda, ldb=ldb, ldc=ldc, config=config)
    assert np.array_equal(C1, C2)
    assert max_err(C1, A, B, C0, si.ALPHA, si.BETA) <= TOL


def test_streamk_integer_bit_exact():
    m, n, k = 900, 700, 1500
    A, B, C0 = si.matrices(m, n, k, 13, kind="integer")
    C, _ = run(A, B, C0, 1.5, 0.5, TF32X3, config="2,128,1")
    R, _ = oracle.sgemm(1.5, A, B, 0.5, C0)
    assert np.array_equal(C.astype(np.float64), R)


@pytest.mark.parametrize("shape", [(1000, 300, 700), (2500, 129, 65), (7, 5, 3)])
@pytest.mark.parametrize("beta", [0.5, 0.0])
def test_sgemm_host_end_to_end(shape, beta):
    """tm_sgemm_host (the e2e leg of bench.py): host buffers with padded
    leading dimensions, row-block copy/compute overlap, result copied back."""
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = shape
    A, B, C0 = si.matrices(m, n, k, seed=sum(shape), lda=k + 3, ldb=n + 1, ldc=n + 2)
    C = np.array(C0.base if C0.base is not None else C0, copy=True)
    Cv = C[:, :n]
    tm.sgemm_host(A, B, Cv, si.ALPHA, beta)
    assert max_err(Cv, A, B, C0, si.ALPHA, beta) <= TOL
    assert np.array_equal(C[:, n:], (C0.base if C0.base is not None else C0)[:, n:])  # padding untouched


@pytest.mark.parametrize("algo", [SIMT, TF32X3])
def test_degenerate_dims(algo):
    """k = 1, n = 1 (tensor-core path with padded ld), m = 1; tall-skinny."""
    for (m, n, k) in [(300, 4, 1), (1, 4, 64), (257, 1, 300), (5000, 8, 32)]:
        pad = lambda x: (x + 3) // 4 * 4
        lda, ldb, ldc = (pad(k), pad(n), pad(n)) if algo == TF32X3 else (k, n, n)
        A, B, C0 = si.matrices(m, n, k, seed=m + k, lda=lda, ldb=ldb, ldc=ldc)
        C, _ = run(A, B, C0, si.ALPHA, si.BETA, algo, lda=lda, ldb=ldb, ldc=ldc)
        assert max_err(C, A, B, C0, si.ALPHA, si.BETA) <= TOL, (m, n, k)


def test_auto_offsets_and_views():
    """AUTO with torch views at element offsets: 16-B aligned sub-views take
    the tensor-core path, misaligned ones fall back to SIMT; both correct."""
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k = 600, 400, 520  # above the small-kernel threshold (m*n*k > 2^24)
    A, B, C0 = si.matrices(m + 4, n + 4, k + 4, seed=99)  # leading dims multiples of 4
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, B, C0))
    assert dA.stride(0) % 4 == 0 and dB.stride(0) % 4 == 0
    for off in (0, 1, 4):
        Av, Bv, Cv = dA[off:off + m - 1, off:off + k - 1], dB[off:off + k - 1, off:off + n - 1], dC.clone()[off:off + m - 1, off:off + n - 1]
        Cref = Cv.cpu().numpy().copy()
        path = tm.plan_name(m - 1, n - 1, k - 1, si.ALPHA, si.BETA, Av.data_ptr(), Av.stride(0), Bv.data_ptr(),
                            Bv.stride(0), Cv.data_ptr(), Cv.stride(0))
        assert path == ("simt" if off % 4 else "tf32x3"), (off, path)
        tm.sgemm(Av, Bv, Cv, si.ALPHA, si.BETA)
        torch.cuda.synchronize()
        An, Bn = Av.cpu().numpy(), Bv.cpu().numpy()
        assert max_err(Cv.cpu().numpy(), An, Bn, Cref, si.ALPHA, si.BETA) <= TOL, off


@pytest.mark.parametrize("algo", [AUTO, TF32X3, 4])  # 4 = BF16X9
def test_random_shape_sweep_sampled_rows(algo):
    """random shapes up to 2048 (log-uniform m, n, k, 60
    draws) through AUTO (every dispatch path: small-GEMM, SIMT, tensor cores,
    stream-K, data-parallel) and forced tensor-core paths; oracle on sampled rows
    (both ends, every 128-row boundary near the tail, seeded random rows)."""
    g = si.rng(2048 + algo)
    for _ in range(60):
        m, n, k = (int(np.exp(g.uniform(0, np.log(2048)))) for _ in range(3))
        pad = lambda x: (x + 3) // 4 * 4
        lda, ldb, ldc = pad(k), pad(n), pad(n)  # aligned, so the forced tensor-core paths accept them
        A, B, C0 = si.matrices(m, n, k, seed=m * 7919 + n * 31 + k, lda=lda, ldb=ldb, ldc=ldc)
        C, _ = run(A, B, C0, si.ALPHA, si.BETA, algo, lda=lda, ldb=ldb, ldc=ldc)
        rows = np.unique(np.concatenate([[0, m - 1], np.arange(max(0, (m // 128) * 128 - 1), m),
                                         g.integers(0, m, 12)]))[:64].astype(np.int64)
        e = max_err(C, A, B, C0, si.ALPHA, si.BETA, rows=rows)
        assert e <= TOL, (m, n, k, e)
