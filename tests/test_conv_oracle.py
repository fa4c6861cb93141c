"""Pins for the convolution oracle (oracle.c: tm_oracle_conv2d_nhwc) --
independent library (numpy einsum over shifted views), the GEMM oracle on an
explicit im2col matrix (sgemm implements convolutions), closed
forms (centred identity filter, all-ones), special cases."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si


def _np_conv(alpha, X, Wt, beta, Y0, pad):
    Nb, H, W, C = X.shape
    F, R, S, _ = Wt.shape
    Xp = np.zeros((Nb, H + 2 * pad, W + 2 * pad, C))
    Xp[:, pad:pad + H, pad:pad + W] = X
    Ho, Wo = H + 2 * pad - R + 1, W + 2 * pad - S + 1
    out = np.zeros((Nb, Ho, Wo, F))
    for ky in range(R):
        for kx in range(S):
            out += np.einsum("bhwc,fc->bhwf", Xp[:, ky:ky + Ho, kx:kx + Wo], Wt[:, ky, kx].astype(np.float64))
    res = alpha * out
    if beta != 0:
        res = res + beta * Y0.astype(np.float64)
    return res.reshape(-1, F)


@pytest.mark.parametrize("shape", [(2, 9, 11, 3, 5, 3, 3, 1), (1, 7, 6, 16, 16, 3, 3, 0), (3, 5, 5, 4, 8, 5, 5, 2),
                                   (1, 12, 10, 2, 3, 1, 1, 0), (2, 8, 8, 16, 16, 7, 7, 3)])
def test_conv_oracle_against_numpy(shape):
    Nb, H, W, C, F, R, S, pad = shape
    g = si.rng(sum(shape))
    X = si.uniform(g, (Nb, H, W, C))
    Wt = si.uniform(g, (F, R, S, C))
    Ho, Wo = H + 2 * pad - R + 1, W + 2 * pad - S + 1
    Y0 = si.uniform(g, (Nb, Ho, Wo, F))
    Rr, Dd = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, pad)
    ref = _np_conv(1.5, X, Wt, 0.5, Y0, pad)
    assert np.max(np.abs(Rr - ref) / Dd) <= 1e-12


def test_conv_equals_gemm_oracle_on_explicit_im2col():
    Nb, H, W, C, F, R, S, pad = 2, 10, 9, 4, 6, 3, 3, 1
    g = si.rng(3)
    X = si.uniform(g, (Nb, H, W, C))
    Wt = si.uniform(g, (F, R, S, C))
    Y0 = si.uniform(g, (Nb, H, W, F))
    Xp = np.zeros((Nb, H + 2, W + 2, C), np.float32)
    Xp[:, 1:H + 1, 1:W + 1] = X
    cols = np.stack([Xp[:, ky:ky + H, kx:kx + W] for ky in range(R) for kx in range(S)], axis=3)  # b,h,w,tap,c
    A = np.ascontiguousarray(cols.reshape(Nb * H * W, R * S * C))            # K index = (ky*S+kx)*C + c
    Bt = np.ascontiguousarray(Wt.reshape(F, R * S * C))                       # KRSC = B^T
    Rg, Dg = oracle.sgemm(1.5, A, Bt, 0.5, Y0.reshape(-1, F), opb="T")
    Rc, Dc = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, pad)
    assert np.array_equal(Rg, Rc) and np.array_equal(Dg, Dc)  # same products, same order


def test_conv_identity_filter_closed_form():
    Nb, H, W, C = 2, 6, 7, 5
    g = si.rng(4)
    X = si.uniform(g, (Nb, H, W, C))
    Wt = np.zeros((C, 3, 3, C), np.float32)
    for c in range(C):
        Wt[c, 1, 1, c] = 1.0                                                   # centred delta: Y = X
    Rr, _ = oracle.conv2d_nhwc(1.0, X, Wt, 0.0, None, 1)
    assert np.array_equal(Rr, X.reshape(-1, C).astype(np.float64))
    ones = np.ones((2, 3, 3, C), np.float32)
    Ro, _ = oracle.conv2d_nhwc(1.0, np.ones((1, 5, 5, C), np.float32), ones, 0.0, None, 0)
    assert np.all(Ro == 9 * C)


def test_conv_pixel_subset_and_special_cases():
    Nb, H, W, C, F = 2, 8, 8, 3, 4
    g = si.rng(5)
    X = si.uniform(g, (Nb, H, W, C))
    Wt = si.uniform(g, (F, 3, 3, C))
    Y0 = si.uniform(g, (Nb, H, W, F))
    Rr, Dd = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, 1)
    pix = np.array([0, 5, 63, 64, 127], np.int64)
    Rs, Ds = oracle.conv2d_nhwc(1.5, X, Wt, 0.5, Y0, 1, pixels=pix)
    assert np.array_equal(Rs, Rr[pix]) and np.array_equal(Ds, Dd[pix])
    Rz, _ = oracle.conv2d_nhwc(0.0, np.full_like(X, np.nan), np.full_like(Wt, np.nan), 0.5, Y0, 1)
    assert np.array_equal(Rz, 0.5 * Y0.reshape(-1, F).astype(np.float64))
    Rb, _ = oracle.conv2d_nhwc(1.5, X, Wt, 0.0, np.full_like(Y0, np.nan), 1)
    assert np.all(np.isfinite(Rb))
