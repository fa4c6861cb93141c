"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no products, no sums of the
GEMM): it only draws random numbers with numpy's PCG64 and lays them out.
Both the oracle (tests, bench cpu_baseline) and the GPU path consume the same
arrays, so parity compares like with like.  Input recipe:

* gating inputs: A, B, C0 ~ U[-1, 1) fp32, alpha = 1.5, beta = 0.5;
* integer-valued variant: entries in {-4..4} (exact in TF32 and fp32);
* stress variant: U[0, 1) (all-positive, non-gating);
* conv (im2col) structure for the skinny config ("sgemm (matrix
  multiplication used to implement convolutions)"): an image X (H x W x Cin)
  ~ U[-1,1), A[(y*W+x), (c*9+ky*3+kx)] = X[y+ky-1, x+kx-1, c] with zero
  padding, weights B (9*Cin x Cout) ~ U[-1,1).
"""
from __future__ import annotations

import numpy as np

ALPHA = 1.5
BETA = 0.5

# BASELINE.json "configs" (index -> (m, n, k)); C3b is the north_star target size.
CONFIGS = {
    "C1": (64, 64, 64),
    "C2": (1060, 1060, 1060),
    "C3": (4096, 4096, 4096),
    "C3b": (8192, 8192, 8192),
    "C4": (50176, 64, 576),
    "C5": (16384, 16384, 16384),
}
SEEDS = {"C1": 1804, "C2": 1805, "C3": 1806, "C3b": 1807, "C4": 1808, "C5": 1809}


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def uniform(g: np.random.Generator, shape, lo=-1.0, hi=1.0) -> np.ndarray:
    """fp32 U[lo, hi): drawn in fp32 directly (no fp64 -> fp32 rounding)."""
    x = g.random(size=shape, dtype=np.float32)
    return (x * np.float32(hi - lo) + np.float32(lo)).astype(np.float32, copy=False)


def integers(g: np.random.Generator, shape, lo=-4, hi=4) -> np.ndarray:
    return g.integers(lo, hi + 1, size=shape).astype(np.float32)


def matrices(m: int, n: int, k: int, seed: int, kind: str = "uniform",
             lda: int | None = None, ldb: int | None = None, ldc: int | None = None):
    """A (m x k), B (k x n), C0 (m x n) float32, optionally padded leading dims.

    With ld* > row length the returned arrays are views into larger buffers,
    so the padding exists in memory (guard band) but is not part of the matrix.
    """
    g = rng(seed)

    def draw(r, c, ld):
        ld = c if ld is None else ld
        if kind == "uniform":
            buf = uniform(g, (r, ld))
        elif kind == "positive":
            buf = uniform(g, (r, ld), 0.0, 1.0)
        elif kind == "integer":
            buf = integers(g, (r, ld))
        else:
            raise ValueError(kind)
        return buf[:, :c]

    A = draw(m, k, lda)
    B = draw(k, n, ldb)
    C0 = draw(m, n, ldc)
    return A, B, C0


def im2col_conv(H: int = 224, W: int = 224, Cin: int = 64, Cout: int = 64, seed: int = 1808):
    """A = im2col(X) (H*W x 9*Cin), B = weights (9*Cin x Cout), C0 (H*W x Cout).

    Column order c*9 + ky*3 + kx, 3x3 window centred on (y, x), zero padding.
    Pure data layout (gathers and zeros), no arithmetic of the GEMM.
    """
    g = rng(seed)
    X = uniform(g, (H, W, Cin))
    Xp = np.zeros((H + 2, W + 2, Cin), dtype=np.float32)
    Xp[1:H + 1, 1:W + 1, :] = X
    A = np.empty((H, W, Cin, 3, 3), dtype=np.float32)
    for ky in range(3):
        for kx in range(3):
            A[:, :, :, ky, kx] = Xp[ky:ky + H, kx:kx + W, :]
    A = A.reshape(H * W, Cin * 9)
    B = uniform(g, (9 * Cin, Cout))
    C0 = uniform(g, (H * W, Cout))
    return A, B, C0


def sample_rows(m: int, count: int = 256, seed: int = 7, tile: int = 128, extra=()) -> np.ndarray:
    """Deterministic row sample: first/last rows, one row per tile band, every
    tile boundary row pair up to ``count``, plus ``extra`` (e.g. shard
    boundaries); sorted and unique."""
    rows = {0, max(m - 1, 0)}
    for b in range(0, m, tile):
        rows.add(b)
        rows.add(min(m - 1, b + tile - 1))
    rows.update(int(r) for r in extra if 0 <= r < m)
    rows = sorted(rows)
    g = rng(seed)
    if len(rows) > count:
        keep = [0, len(rows) - 1] + list(g.choice(np.arange(1, len(rows) - 1), size=count - 2, replace=False))
        rows = sorted(set(rows[i] for i in keep) | {r for r in extra if 0 <= r < m})
    while len(rows) < min(count, m):
        rows = sorted(set(rows) | {int(g.integers(0, m))})
    return np.asarray(rows, dtype=np.int64)


# The paper's image-processing input ("a 2112x3520 RGB input
# image"): the Blur workload runs on it.
BLUR_IMAGE = (2112, 3520)
BLUR_SEED = 1842


def image(N: int, M: int, seed: int = BLUR_SEED, signed: bool = False) -> np.ndarray:
    """N x M x 3 float32 RGB image, channels interleaved (the paper's in[i][j][c]):
    pixel intensities U[0, 1) (or U[-1, 1) with signed=True, a cancellation stress)."""
    return uniform(rng(seed), (N, M, 3), -1.0 if signed else 0.0, 1.0)
