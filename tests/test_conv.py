"""Convolution (tm_conv2d_nhwc, the paper's Conv
benchmark PAPER.md:824-826) against the convolution oracle (pinned in
test_conv_oracle.py): the direct halo-tile tensor-core kernel (default where it
fits), the implicit-GEMM tensor-core kernel (TMA im2col; every compiled
configuration), and the SIMT direct-convolution path."""
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
TOL = 1e-5
TF32X3, SIMT, AUTO = 1, 2, 0


def _run(shape, algo=AUTO, beta=0.5, config=None, seed=0, kind="uniform", path=None):
    import torch
    import paper_1804_10694_b200 as tm
    Nb, H, W, C, F, R, S, pad = shape
    g = si.rng(seed + sum(shape))
    draw = (lambda sh: si.integers(g, sh)) if kind == "integer" else (lambda sh: si.uniform(g, sh))
    X = draw((Nb, H, W, C))
    Wt = draw((F, R, S, C))
    Ho, Wo = H + 2 * pad - R + 1, W + 2 * pad - S + 1
    Y0 = draw((Nb, Ho, Wo, F))
    dX, dW, dY = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (X, Wt, Y0))
    if config:
        os.environ["TM_CONV_CONFIG"] = config
        path = "im2col"
    if path:
        os.environ["TM_CONV_PATH"] = path
    try:
        tm.conv2d_nhwc(dX, dW, dY, 1.5, beta, pad, algo=algo)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("TM_CONV_CONFIG", None)
        os.environ.pop("TM_CONV_PATH", None)
    return X, Wt, Y0, dY.cpu().numpy().reshape(-1, F)


SHAPES = [(2, 9, 11, 16, 16, 3, 3, 1), (1, 7, 6, 16, 16, 3, 3, 0), (2, 13, 10, 32, 64, 3, 5, 2),
          (1, 8, 8, 16, 32, 7, 7, 3), (3, 20, 17, 64, 48, 1, 1, 0), (1, 33, 35, 16, 8, 5, 3, 1)]


@pytest.mark.parametrize("algo,path", [(AUTO, None), (AUTO, "im2col"), (SIMT, None)])
@pytest.mark.parametrize("shape", SHAPES)
def test_conv_parity(algo, path, shape):
    X, Wt, Y0, Y = _run(shape, algo, path=path)
    R, D = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, shape[-1])
    assert float(np.max(oracle.normalized_error(Y, R, D))) <= TOL


@pytest.mark.parametrize("config,shape", [("1,16", (2, 15, 12, 16, 16, 3, 3, 1)), ("1,32", (2, 15, 12, 16, 24, 3, 3, 1)),
                                          ("1,64", (1, 19, 21, 16, 64, 3, 3, 1)), ("2,64", (2, 19, 21, 16, 96, 3, 3, 1)),
                                          ("1,16", (2, 15, 12, 32, 16, 3, 3, 1)), ("1,64", (1, 19, 21, 64, 40, 3, 3, 1)),
                                          ("2,64", (2, 19, 21, 32, 128, 3, 3, 0)), ("2,128", (1, 19, 21, 32, 200, 3, 3, 1))])
def test_conv_tensor_core_configs(config, shape):
    X, Wt, Y0, Y = _run(shape, TF32X3, config=config)
    R, D = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, shape[-1])
    assert float(np.max(oracle.normalized_error(Y, R, D))) <= TOL


# Direct kernel geometry: several 128-pixel tiles per output row with a ragged
# last one, tiles crossing image boundaries, 16/32/48/64 channels (one to
# three halo boxes, 64-B and 128-B swizzled rows), F below / at / above a
# power of two, 1x1 .. 7x7 taps with and without padding, one-pixel rows.
DIRECT_SHAPES = [(2, 6, 300, 16, 16, 3, 3, 1), (3, 5, 128, 16, 16, 3, 3, 1), (1, 4, 257, 32, 32, 3, 3, 1),
                 (2, 5, 140, 48, 20, 3, 3, 1), (1, 4, 130, 64, 64, 3, 3, 1), (2, 7, 150, 16, 8, 5, 5, 2),
                 (2, 6, 131, 16, 40, 1, 1, 0), (1, 9, 200, 32, 16, 3, 5, 0), (2, 3, 1, 16, 16, 3, 3, 1),
                 (1, 40, 3, 16, 12, 3, 1, 1), (1, 9, 140, 16, 16, 3, 7, 3), (2, 6, 133, 16, 24, 5, 5, 2),
                 # 7x7: one TMEM A slot beside two accumulators
                 (2, 20, 150, 16, 16, 7, 7, 3), (1, 12, 133, 16, 12, 7, 7, 0),
                 # even filter widths; 9x9 in passes of filter rows; 11x11 split over kx (two launches)
                 (1, 10, 140, 16, 16, 3, 4, 1), (1, 12, 100, 16, 16, 2, 6, 0), (1, 30, 170, 16, 16, 9, 9, 4),
                 (2, 26, 131, 16, 16, 11, 11, 5), (1, 15, 90, 32, 20, 11, 11, 0)]


@pytest.mark.parametrize("shape", DIRECT_SHAPES)
def test_conv_direct_parity(shape):
    X, Wt, Y0, Y = _run(shape, TF32X3)
    R, D = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, shape[-1])
    assert float(np.max(oracle.normalized_error(Y, R, D))) <= TOL


@pytest.mark.parametrize("path", [None, "im2col"])
def test_conv_beta_zero_and_integer_bit_exact(path):
    shape = (2, 12, 140, 16, 16, 3, 3, 1)
    X, Wt, Y0, Y = _run(shape, TF32X3, beta=0.0, path=path)
    R, D = oracle.conv2d_nhwc(1.5, X, Wt, 0.0, None, 1)
    assert float(np.max(oracle.normalized_error(Y, R, D))) <= TOL
    X, Wt, Y0, Y = _run(shape, TF32X3, kind="integer", path=path)
    R, _ = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, 1)
    assert np.array_equal(Y.astype(np.float64), R)


@pytest.mark.parametrize("path", [None, "im2col"])
def test_conv_paper_shape_sampled_pixels(path):
    """512x512 input, 16 input/output features, batch 32, 3x3."""
    shape = (32, 512, 512, 16, 16, 3, 3, 1)
    X, Wt, Y0, Y = _run(shape, AUTO, seed=1808, path=path)
    P = Y.shape[0]
    g = si.rng(5)
    pix = np.unique(np.concatenate([g.integers(0, P, 3000), [0, 511, 512, 512 * 511, P - 1, P - 512]]))
    R, D = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, 1, pixels=pix)
    assert float(np.max(oracle.normalized_error(Y[pix], R, D))) <= TOL


# The paper's larger specialised filters ("3x3, 5x5, 7x7, 9x9
# and 11x11"), 'same' padding, on the default path (the direct kernel: 9x9 in
# passes, 11x11 in two launches over the filter columns), on the implicit-GEMM
# kernel (TM_CONV_PATH=im2col) and on SIMT; integer inputs bit-exact.
BIG_FILTERS = [(2, 40, 140, 16, 16, 9, 9, 4), (1, 36, 150, 16, 16, 11, 11, 5), (1, 30, 133, 32, 24, 11, 11, 5)]


@pytest.mark.parametrize("algo,path", [(AUTO, None), (AUTO, "im2col"), (SIMT, None)])
@pytest.mark.parametrize("shape", BIG_FILTERS)
def test_conv_9x9_11x11_filters(algo, path, shape):
    X, Wt, Y0, Y = _run(shape, algo, path=path)
    R, D = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, shape[-1])
    assert float(np.max(oracle.normalized_error(Y, R, D))) <= TOL


def test_conv_11x11_integer_bit_exact():
    shape = (1, 24, 140, 16, 16, 11, 11, 5)
    X, Wt, Y0, Y = _run(shape, AUTO, kind="integer")
    R, _ = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, shape[-1])
    assert np.array_equal(Y.astype(np.float64), R)


def test_conv_paper_exact_valid_shape_sampled_pixels():
    """PAPER.md:826 with valid padding: output 510x510,
    the im2col GEMM M = 32*510*510 = 8,323,200, N = 16, K = 144."""
    shape = (32, 512, 512, 16, 16, 3, 3, 0)
    X, Wt, Y0, Y = _run(shape, AUTO, seed=1809)
    P = Y.shape[0]
    assert P == 32 * 510 * 510
    g = si.rng(6)
    pix = np.unique(np.concatenate([g.integers(0, P, 3000), [0, 509, 510, 510 * 509, P - 1, P - 510]]))
    R, D = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, 0, pixels=pix)
    assert float(np.max(oracle.normalized_error(Y[pix], R, D))) <= TOL


def test_conv_simt_fallback_accepts_wide_channels():
    """C = 2576 with F % 4 != 0 misses the tensor-core rule; the SIMT fallback
    tiles the channel dimension through shared memory, so AUTO accepts it."""
    shape = (1, 6, 7, 2576, 18, 3, 3, 1)
    X, Wt, Y0, Y = _run(shape, AUTO)
    R, D = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, 1)
    assert float(np.max(oracle.normalized_error(Y, R, D))) <= TOL
