"""Pins for the blur oracle (oracle.c tm_oracle_blur; the paper's Blur,
PAPER.md:216-219, the workload of its distributed example Fig. 5): a
hand-worked golden case, closed forms (constant image, integer linear ramps),
an independent library (scipy 2-D convolution with a 3x3 box of 1/9), the
tolerance scale, and row-subset consistency."""
import json
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_golden_hand_worked_4x4():
    with open(os.path.join(GOLDEN, "blur_hand_4x4.json")) as f:
        gold = json.load(f)
    img = np.array(gold["in"], dtype=np.float32)
    R, D = oracle.blur(img)
    assert np.array_equal(R, np.array(gold["by"], dtype=np.float64))
    assert np.array_equal(D, R)  # non-negative inputs


def test_constant_image():
    img = np.full((9, 14, 3), 2.5, dtype=np.float32)
    R, D = oracle.blur(img)
    assert R.shape == (7, 12, 3) and np.all(R == 2.5) and np.all(D == 2.5)


@pytest.mark.parametrize("a,b,c0", [(3, -2, 7), (0, 5, -4), (-7, 1, 0)])
def test_integer_linear_ramp_is_its_centre_value(a, b, c0):
    N, M = 11, 17
    i, j = np.meshgrid(np.arange(N), np.arange(M), indexing="ij")
    ramp = (a * i + b * j + c0).astype(np.float32)
    img = np.stack([ramp, -ramp, 2 * ramp], axis=-1)
    R, _ = oracle.blur(img)
    centre = (a * (i[:-2, :-2] + 1) + b * (j[:-2, :-2] + 1) + c0).astype(np.float64)
    assert np.array_equal(R[..., 0], centre)
    assert np.array_equal(R[..., 1], -centre)
    assert np.array_equal(R[..., 2], 2 * centre)


@pytest.mark.parametrize("shape", [(3, 3), (5, 40), (64, 33), (130, 7)])
def test_against_scipy_convolution(shape):
    from scipy.signal import convolve2d
    N, M = shape
    img = si.uniform(si.rng(N * 31 + M), (N, M, 3))
    R, D = oracle.blur(img)
    box = np.full((3, 3), 1.0 / 9.0)
    for c in range(3):
        x = img[..., c].astype(np.float64)
        ref = convolve2d(x, box, mode="valid")
        assert np.max(np.abs(R[..., c] - ref) / convolve2d(np.abs(x), box, mode="valid")) <= 1e-14
        assert np.allclose(D[..., c], convolve2d(np.abs(x), box, mode="valid"), rtol=1e-14, atol=0)


def test_row_subset_and_invalid():
    img = si.uniform(si.rng(3), (40, 25, 3))
    R, D = oracle.blur(img)
    rows = np.array([0, 5, 37], dtype=np.int64)
    Rs, Ds = oracle.blur(img, rows=rows)
    assert np.array_equal(Rs, R[rows]) and np.array_equal(Ds, D[rows])
    with pytest.raises(ValueError):
        oracle.blur(np.zeros((2, 5, 3), np.float32))
