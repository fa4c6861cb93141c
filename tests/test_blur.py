"""GPU parity of the blur (tm_blur, tm_blur_dist_loopback; the paper's Blur,
PAPER.md:216-219, and its row-distributed schedule, Fig. 5 Code 3,
PAPER.md:494-557) against the oracle (oracle.c tm_oracle_blur), element by
element.

Tolerance: the kernel computes in fp32 with "/3"
as a multiply by fl(1/3): bx = fl(fl(fl(a+b)+e) * t), by likewise over three
bx.  Every rounding is at most u = 2^-24 relative to a partial whose magnitude
is bounded by the sum of |in| it covers, so |by - R| <= ~8u * D with D the
mean |in| over the nine taps (the oracle's D); the gate is 1e-6 * D (about
16u), and D == 0 requires exact zeros.
"""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
TOL = 1e-6


def _err(out, R, D):
    out = out.astype(np.float64)
    diff = np.abs(out - R)
    if np.any((D == 0) & (diff != 0)):
        return np.inf
    with np.errstate(divide="ignore", invalid="ignore"):
        e = np.where(D == 0, 0.0, diff / np.where(D == 0, 1.0, D))
    return float(e.max()) if e.size else 0.0


def _dev_image(img, ld=None, offset=0, fill=-777.0):
    """Device copy of an (N, M, 3) image with row pitch ld (>= 3M) floats,
    starting `offset` floats into its buffer (offset 1: a 4-byte misaligned
    base); returns the (N, M, 3) view."""
    import torch
    N, M, _ = img.shape
    ld = 3 * M if ld is None else ld
    buf = torch.full((offset + N * ld + 8,), fill, dtype=torch.float32, device="cuda")
    v = buf[offset:offset + N * ld].view(N, ld)[:, :3 * M]
    v.copy_(torch.from_numpy(img.reshape(N, 3 * M)))
    return v.view(N, M, 3), buf


def _dev_out(N, M, ld=None, offset=0, fill=-555.0):
    import torch
    ld = 3 * M if ld is None else ld
    buf = torch.full((offset + N * ld + 8,), fill, dtype=torch.float32, device="cuda")
    return buf[offset:offset + N * ld].view(N, ld)[:, :3 * M].view(N, M, 3), buf


@pytest.mark.parametrize("N,M", [(3, 3), (4, 4), (5, 7), (33, 3), (64, 33), (130, 7), (257, 1000), (1000, 45),
                                 (67, 2051)])
def test_blur_dense(N, M):
    import torch
    import paper_1804_10694_b200 as tm
    img = si.image(N, M, seed=N * 7919 + M)
    R, D = oracle.blur(img)
    dIn, _ = _dev_image(img)
    out = tm.blur(dIn)
    torch.cuda.synchronize()
    assert _err(out.cpu().numpy(), R, D) <= TOL


@pytest.mark.parametrize("ldi_pad,ldo_pad,ioff,ooff", [
    (0, 0, 1, 0),      # misaligned input base: scalar loads
    (0, 0, 0, 1),      # misaligned output base: scalar stores
    (4, 4, 0, 0),      # padded pitches, both 16-B aligned rows
    (1, 3, 0, 2),      # odd pitches, 8-B aligned output base
    (12, 2, 0, 0),     # even output pitch: float2 stores
])
def test_blur_pitch_and_alignment(ldi_pad, ldo_pad, ioff, ooff):
    import torch
    import paper_1804_10694_b200 as tm
    N, M = 97, 130
    img = si.image(N, M, seed=5, signed=True)
    R, D = oracle.blur(img)
    dIn, _ = _dev_image(img, 3 * M + ldi_pad, ioff)
    dOut, obuf = _dev_out(N - 2, M - 2, 3 * (M - 2) + ldo_pad, ooff)
    tm.blur(dIn, dOut)
    torch.cuda.synchronize()
    assert _err(dOut.cpu().numpy(), R, D) <= TOL
    # nothing outside the output view was written (guard band and row padding)
    b = obuf.cpu().numpy()
    mask = np.ones(b.shape, bool)
    ld = 3 * (M - 2) + ldo_pad
    for i in range(N - 2):
        mask[ooff + i * ld: ooff + i * ld + 3 * (M - 2)] = False
    assert np.all(b[mask] == np.float32(-555.0))


def test_blur_zero_and_constant_images():
    import torch
    import paper_1804_10694_b200 as tm
    z = torch.zeros((40, 50, 3), device="cuda")
    assert torch.count_nonzero(tm.blur(z)) == 0
    c = torch.full((40, 50, 3), 0.75, device="cuda")
    o = tm.blur(c)
    torch.cuda.synchronize()
    # (3 * 0.75) * fl(1/3) twice: within one ulp chain of 0.75
    assert float((o - 0.75).abs().max()) <= 4 * 2.0 ** -24


def test_blur_paper_image_sampled_rows():
    """The paper's 2112x3520 RGB image in the launch
    configuration bench.py times; oracle on sampled rows covering every
    32-row strip boundary and the image edges."""
    import torch
    import paper_1804_10694_b200 as tm
    N, M = si.BLUR_IMAGE
    img = si.image(N, M)
    dIn, _ = _dev_image(img)
    out = tm.blur(dIn)
    torch.cuda.synchronize()
    rows = sorted({0, 1, N - 4, N - 3} | {r for s in range(0, N - 2, 32) for r in (s, s + 31) if r < N - 2}
                  | set(si.rng(9).integers(0, N - 2, 40).tolist()))
    rows = np.array(rows, dtype=np.int64)
    R, D = oracle.blur(img, rows=rows)
    assert _err(out.cpu().numpy()[rows], R, D) <= TOL


def test_blur_deterministic():
    import torch
    import paper_1804_10694_b200 as tm
    img = torch.from_numpy(si.image(300, 301, seed=3)).cuda()
    a, b = tm.blur(img), tm.blur(img)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("P,N,M", [(2, 9, 11), (3, 50, 40), (4, 101, 37), (8, 2112, 64), (8, 18, 5), (5, 23, 300)])
def test_blur_dist_loopback(P, N, M):
    """Each simulated rank holds its chunk plus the 2-row border region; rank r's
    border comes from rank r+1; every rank's output rows
    match the oracle's rows [row0, row0+rows), and each rank but the last
    receives exactly two rows (ldi + 3M floats)."""
    import torch
    import paper_1804_10694_b200 as tm
    img = si.image(N, M, seed=P * 1000 + N, signed=True)
    R, D = oracle.blur(img)
    lins, louts, parts = [], [], []
    for r in range(P):
        r0, rows = tm.dist_rows(N - 2, P, r)
        lin = torch.full((rows + 2, M, 3), float("nan"), device="cuda")
        lin[:rows] = torch.from_numpy(img[r0:r0 + rows]).cuda()
        if r == P - 1:
            lin[rows:] = torch.from_numpy(img[N - 2:]).cuda()
        lins.append(lin)
        louts.append(torch.full((rows, M - 2, 3), float("nan"), device="cuda"))
        parts.append((r0, rows))
    got = tm.blur_dist_loopback(N, M, lins, louts)
    torch.cuda.synchronize()
    for r, (r0, rows) in enumerate(parts):
        assert _err(louts[r].cpu().numpy(), R[r0:r0 + rows], D[r0:r0 + rows]) <= TOL, r
        assert got[r] == (0 if r == P - 1 else (3 * M + 3 * M) * 4)
        if r < P - 1:  # the received border rows are rank r+1's first two rows
            assert np.array_equal(lins[r][rows:].cpu().numpy(), img[r0 + rows:r0 + rows + 2])
    # single-GPU tm_blur gives the same bits (same kernel, same strips per row)
    full = tm.blur(torch.from_numpy(img).cuda())
    torch.cuda.synchronize()
    ref = full.cpu().numpy()
    for r, (r0, rows) in enumerate(parts):
        assert np.array_equal(louts[r].cpu().numpy(), ref[r0:r0 + rows])


def test_blur_dist_rejects_too_many_ranks():
    import torch
    import paper_1804_10694_b200 as tm
    N, M, P = 9, 6, 4  # (N-2)/P = 1 < 2: a chunk cannot supply two border rows
    lins = [torch.zeros((tm.dist_rows(N - 2, P, r)[1] + 2, M, 3), device="cuda") for r in range(P)]
    louts = [torch.zeros((tm.dist_rows(N - 2, P, r)[1], M - 2, 3), device="cuda") for r in range(P)]
    with pytest.raises(tm.TmError):
        tm.blur_dist_loopback(N, M, lins, louts)


@pytest.mark.parametrize("N,M", [(3, 3), (3, 200), (200, 3), (4, 5)])
def test_blur_minimal_images(N, M):
    """The smallest images of the iteration domain i < N-2, j < M-2:
    a single output row, a single output column, a 2x3 output."""
    import torch
    import paper_1804_10694_b200 as tm
    img = si.image(N, M, seed=N + 17 * M, signed=True)
    R, D = oracle.blur(img)
    out = tm.blur(torch.from_numpy(img).cuda())
    torch.cuda.synchronize()
    assert out.shape == (N - 2, M - 2, 3)
    assert _err(out.cpu().numpy(), R, D) <= TOL


def test_blur_dist_loopback_maximum_ranks():
    """(N-2)/P == 2: every chunk is exactly the two border rows its upper
    neighbour needs (the tightest distribution the schedule accepts)."""
    import torch
    import paper_1804_10694_b200 as tm
    P, N, M = 6, 14, 50
    img = si.image(N, M, seed=99)
    R, D = oracle.blur(img)
    lins, louts = [], []
    for r in range(P):
        r0, rows = tm.dist_rows(N - 2, P, r)
        assert rows == 2
        lin = torch.from_numpy(np.ascontiguousarray(img[r0:r0 + rows + 2])).cuda()
        if r < P - 1:
            lin[rows:] = float("nan")
        lins.append(lin)
        louts.append(torch.empty((rows, M - 2, 3), device="cuda"))
    tm.blur_dist_loopback(N, M, lins, louts)
    torch.cuda.synchronize()
    got = torch.cat(louts).cpu().numpy()
    assert _err(got, R, D) <= TOL
