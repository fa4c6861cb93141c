"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each test names what fixes the expected value: exact rational arithmetic
(brute force), an independent library (numpy float64 matmul, numpy int64
matmul), closed forms, the hand-worked golden fixture, and invariants.
Chosen so that a dropped term, a wrong sign or index, or a transposed operand
in the oracle fails at least one of them (see test_pins_catch_mutations).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import seeded_inputs as si

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EPS53 = 2.0 ** -53


def _exact(alpha, A, B, beta, C0):
    """Exact rational R and D (brute force, PAPER.md:67 definition)."""
    m, k = A.shape
    n = B.shape[1]
    R = [[None] * n for _ in range(m)]
    D = [[None] * n for _ in range(m)]
    fa, fb = Fraction(float(alpha)), Fraction(float(beta))
    for i in range(m):
        for j in range(n):
            s = sum((Fraction(float(A[i, p])) * Fraction(float(B[p, j])) for p in range(k)), Fraction(0))
            sa = sum((abs(Fraction(float(A[i, p])) * Fraction(float(B[p, j]))) for p in range(k)), Fraction(0))
            c = Fraction(float(C0[i, j]))
            R[i][j] = fa * s + fb * c
            D[i][j] = abs(fa) * sa + abs(fb) * abs(c)
    return R, D


def test_brute_force_exact_rationals_all_small_shapes():
    g = si.rng(11)
    for m in range(1, 7):
        for n in range(1, 7):
            for k in range(1, 7):
                A = si.uniform(g, (m, k))
                B = si.uniform(g, (k, n))
                C0 = si.uniform(g, (m, n))
                alpha, beta = np.float32(1.5), np.float32(-0.75)
                R, D = oracle.sgemm(alpha, A, B, beta, C0)
                Rx, Dx = _exact(alpha, A, B, beta, C0)
                for i in range(m):
                    for j in range(n):
                        bound = (k + 3) * EPS53 * float(Dx[i][j])
                        assert abs(Fraction(R[i, j]) - Rx[i][j]) <= Fraction(bound), (m, n, k, i, j)
                        assert abs(Fraction(D[i, j]) - Dx[i][j]) <= Fraction(bound), (m, n, k, i, j)


def test_golden_hand_worked_example():
    with open(os.path.join(GOLDEN, "gemm_hand_2x3x2.json")) as f:
        gold = json.load(f)
    A = np.array(gold["A"], dtype=np.float32)
    B = np.array(gold["B"], dtype=np.float32)
    C0 = np.array(gold["C0"], dtype=np.float32)
    R, D = oracle.sgemm(gold["alpha"], A, B, gold["beta"], C0)
    assert np.array_equal(R, np.array(gold["C"], dtype=np.float64))
    assert np.array_equal(D, np.array(gold["D"], dtype=np.float64))


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 13, 5), (64, 64, 64), (129, 65, 257), (200, 31, 96)])
def test_against_numpy_float64_matmul(m, n, k):
    A, B, C0 = si.matrices(m, n, k, seed=m * 7 + n * 3 + k, lda=k + 3, ldb=n + 5, ldc=n + 1)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    A64, B64, C64 = (x.astype(np.float64) for x in (A, B, C0))
    Rn = si.ALPHA * (A64 @ B64) + si.BETA * C64
    Dn = si.ALPHA * (np.abs(A64) @ np.abs(B64)) + si.BETA * np.abs(C64)
    assert np.max(np.abs(R - Rn) / Dn) <= 1e-12
    assert np.max(np.abs(D - Dn) / Dn) <= 1e-12


def test_integer_inputs_exact_against_int64_matmul():
    m, n, k = 97, 83, 301
    A, B, C0 = si.matrices(m, n, k, seed=5, kind="integer")
    R, _ = oracle.sgemm(1.5, A, B, 0.5, C0)
    Ai, Bi, Ci = (x.astype(np.int64) for x in (A, B, C0))
    # 1.5*x + 0.5*c = (3x + c)/2, exact in int64 then one exact division by 2
    expect = (3 * (Ai @ Bi) + Ci).astype(np.float64) / 2.0
    assert np.array_equal(R, expect)


def test_identity_closed_form():
    n = 37
    g = si.rng(3)
    B = si.uniform(g, (n, 19))
    C0 = si.uniform(g, (n, 19))
    eye = np.eye(n, dtype=np.float32)
    R, _ = oracle.sgemm(1.5, eye, B, 0.5, C0)
    assert np.array_equal(R, 1.5 * B.astype(np.float64) + 0.5 * C0.astype(np.float64))


def test_permutation_closed_form():
    n = 41
    g = si.rng(4)
    perm = g.permutation(n)
    P = np.zeros((n, n), dtype=np.float32)
    P[np.arange(n), perm] = 1.0  # (P B)[i,:] = B[perm[i], :]
    B = si.uniform(g, (n, 23))
    R, _ = oracle.sgemm(1.0, P, B, 0.0, None)
    assert np.array_equal(R, B[perm].astype(np.float64))


def test_all_ones_closed_form():
    m, n, k = 9, 11, 1000
    A = np.ones((m, k), dtype=np.float32)
    B = np.ones((k, n), dtype=np.float32)
    C0 = np.full((m, n), 3.0, dtype=np.float32)
    R, D = oracle.sgemm(1.5, A, B, 0.5, C0)
    assert np.all(R == 1.5 * k + 1.5)
    assert np.all(D == 1.5 * k + 1.5)


def test_alpha_zero_does_not_read_A_B():
    m, n, k = 5, 6, 7
    A = np.full((m, k), np.nan, dtype=np.float32)
    B = np.full((k, n), np.nan, dtype=np.float32)
    g = si.rng(9)
    C0 = si.uniform(g, (m, n))
    R, D = oracle.sgemm(0.0, A, B, 0.5, C0)
    assert np.array_equal(R, 0.5 * C0.astype(np.float64))
    assert np.array_equal(D, 0.5 * np.abs(C0.astype(np.float64)))
    R2, _ = oracle.sgemm(0.0, None, None, 0.5, C0, m=m, n=n, k=k)
    assert np.array_equal(R, R2)


def test_beta_zero_does_not_read_C():
    m, n, k = 5, 6, 7
    g = si.rng(10)
    A = si.uniform(g, (m, k))
    B = si.uniform(g, (k, n))
    C0 = np.full((m, n), np.nan, dtype=np.float32)
    R, D = oracle.sgemm(2.0, A, B, 0.0, C0)
    assert np.all(np.isfinite(R)) and np.all(np.isfinite(D))
    assert np.allclose(R, 2.0 * (A.astype(np.float64) @ B.astype(np.float64)), rtol=0, atol=1e-12)


def test_k_zero_is_beta_scale_and_both_zero_is_zero():
    m, n = 4, 3
    g = si.rng(12)
    C0 = si.uniform(g, (m, n))
    R, _ = oracle.sgemm(1.5, None, None, 0.5, C0, m=m, n=n, k=0)
    assert np.array_equal(R, 0.5 * C0.astype(np.float64))
    R0, D0 = oracle.sgemm(0.0, None, None, 0.0, None, m=m, n=n, k=5)
    assert np.array_equal(R0, np.zeros((m, n))) and np.array_equal(D0, np.zeros((m, n)))


def test_empty_shapes():
    R, D = oracle.sgemm(1.0, np.zeros((0, 4), np.float32), np.zeros((4, 3), np.float32), 0.0, None)
    assert R.shape == (0, 3)
    R, D = oracle.sgemm(1.0, np.zeros((2, 4), np.float32), np.zeros((4, 0), np.float32), 0.0, None)
    assert R.shape == (2, 0)


def test_row_subset_matches_full_rows():
    m, n, k = 300, 70, 90
    A, B, C0 = si.matrices(m, n, k, seed=21)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    rows = si.sample_rows(m, count=40, tile=128)
    Rs, Ds = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, rows=rows)
    assert np.array_equal(Rs, R[rows]) and np.array_equal(Ds, D[rows])


def test_thread_count_invariance():
    m, n, k = 257, 129, 200
    A, B, C0 = si.matrices(m, n, k, seed=22)
    t0 = oracle.get_threads()
    try:
        oracle.set_threads(1)
        R1, D1 = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
        oracle.set_threads(max(2, os.cpu_count() or 2))
        R2, D2 = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    finally:
        oracle.set_threads(t0)
    assert np.array_equal(R1, R2) and np.array_equal(D1, D2)


def test_invalid_arguments_rejected():
    A = np.zeros((3, 4), np.float32)
    B = np.zeros((4, 5), np.float32)
    C = np.zeros((3, 5), np.float32)
    with pytest.raises(ValueError):
        oracle.sgemm(1.0, A, B, 1.0, C, m=-1)
    with pytest.raises(ValueError):
        oracle.sgemm(1.0, None, B, 1.0, C, m=3, k=4)  # alpha != 0 needs A
    with pytest.raises(ValueError):
        oracle.sgemm(1.0, A, B, 1.0, None, n=5)  # beta != 0 needs C0


def test_golden_tiling_map_and_partition():
    """PAPER.md:753-758 tiling map (golden) and the row partition that
    generalises split(i, N/Ranks) to P not dividing m."""
    with open(os.path.join(GOLDEN, "tiling_map_32.json")) as f:
        gold = json.load(f)
    T = gold["tile"]
    for ex in gold["examples"]:
        assert ex["i"] // T == ex["i0"] and ex["i"] % T == ex["i1"]
    assert -(-gold["N"] // T) == gold["tiles_per_dim"]
    assert gold["N"] - (gold["tiles_per_dim"] - 1) * T == gold["partial_tile_extent"]
    for m in [0, 1, 7, 16, 1060, 16384, 16385]:
        for P in [1, 2, 3, 4, 8]:
            parts = [oracle.dist_rows(m, P, r) for r in range(P)]
            covered = []
            for r0, nr in parts:
                covered.extend(range(r0, r0 + nr))
            assert covered == list(range(m))  # every row exactly once, in rank order
            assert max(nr for _, nr in parts) - min(nr for _, nr in parts) <= 1
            if m % P == 0:
                assert all(p == (r * (m // P), m // P) for r, p in enumerate(parts))


def test_normalized_error_metric():
    R = np.array([[1.0, 0.0, 2.0]])
    D = np.array([[2.0, 0.0, 4.0]])
    C = np.array([[1.5, 0.0, 2.0]], dtype=np.float32)
    err = oracle.normalized_error(C, R, D)
    assert err[0, 0] == 0.25 and err[0, 1] == 0.0 and err[0, 2] == 0.0
    assert np.isinf(oracle.normalized_error(np.array([[1e-30]], np.float32), np.array([[0.0]]), np.array([[0.0]])))[0, 0]
    assert np.isinf(oracle.normalized_error(np.array([[np.nan]], np.float32), R[:, :1], D[:, :1]))[0, 0]


def test_golden_dist_rows_uneven_partition():
    """Hand-worked partitions (tests/golden/dist_rows.json, PAPER.md:503-504
    split(i, N/Ranks), generalised per SURVEY.md 8(b)): the m mod P extra rows
    go to the first ranks."""
    with open(os.path.join(GOLDEN, "dist_rows.json")) as f:
        gold = json.load(f)
    for case in gold["cases"]:
        got = [list(oracle.dist_rows(case["m"], case["P"], r)) for r in range(case["P"])]
        assert got == case["parts"], (case["m"], case["P"], got)


@pytest.mark.parametrize("opa,opb", [("N", "T"), ("T", "N"), ("T", "T")])
def test_transposed_operands_pins(opa, opb):
    """op(A), op(B) only change where elements are read: the oracle on
    transposed storage must equal the NN oracle on explicit transposed copies
    bit for bit (same products, same summation order), and exact rationals on
    tiny shapes."""
    m, n, k = 37, 23, 29
    A, B, C0 = si.matrices(m, n, k, seed=71)
    At = np.ascontiguousarray(A.T) if opa == "T" else A
    Bt = np.ascontiguousarray(B.T) if opb == "T" else B
    R0, D0 = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    R1, D1 = oracle.sgemm(si.ALPHA, At, Bt, si.BETA, C0, opa=opa, opb=opb)
    assert np.array_equal(R0, R1) and np.array_equal(D0, D1)
    # padded leading dimensions on the transposed storage
    Ap = np.zeros((At.shape[0], At.shape[1] + 5), np.float32)
    Ap[:, :At.shape[1]] = At
    Bp = np.zeros((Bt.shape[0], Bt.shape[1] + 3), np.float32)
    Bp[:, :Bt.shape[1]] = Bt
    R2, _ = oracle.sgemm(si.ALPHA, Ap[:, :At.shape[1]], Bp[:, :Bt.shape[1]], si.BETA, C0, opa=opa, opb=opb)
    assert np.array_equal(R0, R2)
    g = si.rng(72)
    for (mm, nn, kk) in [(2, 3, 4), (3, 1, 2), (1, 4, 3)]:
        a, b, c = si.uniform(g, (mm, kk)), si.uniform(g, (kk, nn)), si.uniform(g, (mm, nn))
        at = np.ascontiguousarray(a.T) if opa == "T" else a
        bt = np.ascontiguousarray(b.T) if opb == "T" else b
        R, _ = oracle.sgemm(1.5, at, bt, -0.75, c, opa=opa, opb=opb)
        Rx, Dx = _exact(1.5, a, b, -0.75, c)
        for i in range(mm):
            for j in range(nn):
                assert abs(Fraction(R[i, j]) - Rx[i][j]) <= Fraction((kk + 3) * EPS53 * float(Dx[i][j]))
