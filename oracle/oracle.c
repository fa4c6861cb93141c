/*
 * oracle.c -- CPU ORACLE FOR THE tm_sgemm HOT PATH.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load or execute this file.  The product library
 * (paper_1804_10694_b200/, include/tm.h) never links, includes or calls it, and
 * this file includes nothing from the product: the two share no code.
 *
 * What it computes (SI "Introduction"):
 *
 *     C = alpha * A * B + beta * C
 *
 * written out as its plain definition, in fp64, no blocking, no fusion, no
 * reordering beyond the definition:
 *
 *     R[i,j] = alpha * sum_{p=0}^{k-1} A[i,p] * B[p,j]  +  beta * C0[i,j]
 *     D[i,j] = |alpha| * sum_{p=0}^{k-1} |A[i,p]| * |B[p,j]|  +  |beta| * |C0[i,j]|
 *
 * D is the denominator of the acceptance metric of BASELINE.json north_star:
 *     err[i,j] = |C_gpu[i,j] - R[i,j]| / D[i,j]  <= 1e-5.
 *
 * Readings of points the paper leaves open:
 *   - storage is row-major (reading 1): A[i*lda+p], B[p*ldb+j], C0[i*ldc+j];
 *   - transposed operands (BLAS op(A), op(B), not in the
 *     paper, whose gemm has none, reading 2) only change WHERE element (i,p) of
 *     A and (p,j) of B are read: opA = T reads A[p*lda+i], opB = T reads
 *     B[j*ldb+p]; the products and their summation order are unchanged;
 *   - special cases follow reference-BLAS semantics (reading 5):
 *       beta == 0          -> C0 is NOT read (NaN in C0 does not propagate);
 *       alpha == 0 or k==0 -> A and B are NOT read, R = beta*C0;
 *       m == 0 or n == 0   -> nothing is computed.
 *
 * Arithmetic: every product of two fp32 values is exact in fp64 (24+24 < 53
 * significand bits); the sum over p runs in the order p = 0..k-1 for every
 * (i,j), i.e. the textbook i-j-p loop's order.  The i-p-j loop order below
 * (a row accumulator acc[0..n)) performs, for each element, exactly the same
 * fp64 operations in the same order, so it is bit-identical to the i-j-p loop;
 * it is used only because it reads B row-wise.  OpenMP parallelises over rows
 * i, which are independent: results do not depend on the thread count.
 *
 * Errors: returns 0 on success, -1 on invalid arguments (negative sizes,
 * leading dimensions smaller than the row length, NULL pointers that would be
 * read), -2 if the row accumulator cannot be allocated.  Outputs are not
 * touched on error.
 *
 * Pins: tests/test_oracle.py checks this file against exact rational
 * arithmetic (brute force, all m,n,k in [1,6]), numpy's float64 matmul,
 * closed forms (identity, permutation, all-ones, alpha=0, beta=0 with NaN
 * poison), integer-valued inputs, and a hand-computed golden example
 * (tests/golden/).
 *
 * The other functions of this file, each with its own header below and its
 * own pins: tm_oracle_conv2d_nhwc (the convolution of PAPER.md:824-826;
 * tests/test_conv_oracle.py), tm_oracle_dist_rows (the row partition,
 * PAPER.md:503-504; tests/golden/dist_rows.json), tm_oracle_blur (the Blur of
 * PAPER.md:216-219; tests/test_blur_oracle.py, tests/golden/blur_hand_4x4.json).
 * tests/test_oracle_mutants.py rebuilds this file with each ORACLE_MUTANT and
 * requires every mutant to fail a pin.  Every function is pinned.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Mutation testing of the pins (tests/test_oracle_mutants.py): a build with
 * -DORACLE_MUTANT=n breaks exactly one step on purpose, and the pin suite must
 * then fail.  The shipped build is ORACLE_MUTANT == 0, where every MUT(n) is the
 * constant 0 and the code below is the plain definition.
 *    1 beta term dropped from R          7 alpha dropped from R
 *    2 last product (p = k-1) dropped    8 conv: filter taps flipped (convolution vs correlation)
 *    3 op(B) read transposed             9 conv: padding not subtracted from the input row
 *    4 lda ignored (A read as dense)    10 dist_rows: the m mod P extra rows go to the LAST ranks
 *    5 fabs dropped from D              11 beta == 0 still reads C0
 *    6 beta term subtracted             12 blur: bx reads in(i, j+1) instead of in(i, j+2)
 *                                       13 blur: by's average misses its /3 */
#ifndef ORACLE_MUTANT
#define ORACLE_MUTANT 0
#endif
#define MUT(n) (ORACLE_MUTANT == (n))

static int64_t max1(int64_t x) { return x > 1 ? x : 1; }

static int check_args(int opa, int opb, int64_t m, int64_t n, int64_t k, float alpha,
                      const float *A, int64_t lda, const float *B, int64_t ldb,
                      float beta, const float *C0, int64_t ldc) {
    if (m < 0 || n < 0 || k < 0) return -1;
    if ((opa != 0 && opa != 1) || (opb != 0 && opb != 1)) return -1;
    int reads_ab = (alpha != 0.0f) && (k > 0);
    if (reads_ab) {
        if (!A || !B) return -1;
        if (lda < (opa ? max1(m) : max1(k))) return -1;
        if (ldb < (opb ? max1(k) : max1(n))) return -1;
    }
    if (beta != 0.0f) {
        if (!C0) return -1;
        if (ldc < (n > 1 ? n : 1)) return -1;
    }
    return 0;
}

/* One output row i of the definition above, into R_row[0..n), D_row[0..n).
 * acc/acc_abs are caller-provided scratch of n doubles each. */
static void oracle_row(int opa, int opb, int64_t i, int64_t n, int64_t k, float alpha,
                       const float *A, int64_t lda, const float *B, int64_t ldb,
                       float beta, const float *C0, int64_t ldc,
                       double *R_row, double *D_row, double *acc, double *acc_abs) {
    const double a_alpha = (double)alpha;
    const double a_beta = (double)beta;
    for (int64_t j = 0; j < n; ++j) { acc[j] = 0.0; acc_abs[j] = 0.0; }
    if (alpha != 0.0f) {
        for (int64_t p = 0; p < k - MUT(2); ++p) {
            const double a = (double)(opa ? A[p * lda + i] : A[i * (MUT(4) ? k : lda) + p]);   /* op(A)[i,p] */
            const double a_abs = MUT(5) ? a : fabs(a);
            for (int64_t j = 0; j < n; ++j) {
                const double b = (double)((opb ^ MUT(3)) ? B[j * ldb + p] : B[p * ldb + j]); /* op(B)[p,j] */
                acc[j] += a * b;             /* exact product, fp64 sum, p ascending */
                acc_abs[j] += a_abs * (MUT(5) ? b : fabs(b));
            }
        }
    }
    for (int64_t j = 0; j < n; ++j) {
        double r = 0.0, d = 0.0;
        if (alpha != 0.0f) {
            r = (MUT(7) ? 1.0 : a_alpha) * acc[j];
            d = fabs(a_alpha) * acc_abs[j];
        }
        if (beta != 0.0f || (MUT(11) && C0)) {   /* beta == 0: C0 is not read */
            const double c = (double)C0[i * ldc + j];
            r += (MUT(6) ? -a_beta : MUT(1) ? 0.0 : a_beta) * c;
            d += fabs(a_beta) * fabs(c);
        }
        R_row[j] = r;
        D_row[j] = d;
    }
}

/* Rows rows[0..nrows) of R and D for C = alpha*op(A)*op(B) + beta*C0 (row t of
 * the outputs is row rows[t] of C); opa/opb: 0 = N, 1 = T.  rows == NULL means
 * all rows 0..m-1 (nrows must then equal m).  R, D are nrows x n, row-major
 * with leading dimension ldr >= n. */
int tm_oracle_sgemm_op_rows(int opa, int opb, int64_t m, int64_t n, int64_t k, float alpha,
                            const float *A, int64_t lda, const float *B, int64_t ldb,
                            float beta, const float *C0, int64_t ldc,
                            int64_t nrows, const int64_t *rows,
                            double *R, double *D, int64_t ldr) {
    if (check_args(opa, opb, m, n, k, alpha, A, lda, B, ldb, beta, C0, ldc)) return -1;
    if (nrows < 0 || ldr < n || (nrows > 0 && (!R || !D))) return -1;
    if (!rows && nrows != m) return -1;
    if (rows)
        for (int64_t t = 0; t < nrows; ++t)
            if (rows[t] < 0 || rows[t] >= m) return -1;
    if (nrows == 0 || n == 0) return 0;
    if (k == 0) alpha = 0.0f;             /* empty sum: A and B are not read */
    int failed = 0;
#pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)n);
        double *acc_abs = (double *)malloc(sizeof(double) * (size_t)n);
        if (!acc || !acc_abs) {
#pragma omp atomic write
            failed = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t t = 0; t < nrows; ++t) {
                const int64_t i = rows ? rows[t] : t;
                oracle_row(opa, opb, i, n, k, alpha, A, lda, B, ldb, beta, C0, ldc,
                           R + t * ldr, D + t * ldr, acc, acc_abs);
            }
        }
        free(acc);
        free(acc_abs);
    }
    return failed ? -2 : 0;
}

/* No transposes (the paper's gemm). */
int tm_oracle_sgemm_rows(int64_t m, int64_t n, int64_t k, float alpha,
                         const float *A, int64_t lda, const float *B, int64_t ldb,
                         float beta, const float *C0, int64_t ldc,
                         int64_t nrows, const int64_t *rows,
                         double *R, double *D, int64_t ldr) {
    return tm_oracle_sgemm_op_rows(0, 0, m, n, k, alpha, A, lda, B, ldb, beta, C0, ldc,
                                   nrows, rows, R, D, ldr);
}

/* All rows: R, D are m x n with leading dimension ldr. */
int tm_oracle_sgemm_f64(int64_t m, int64_t n, int64_t k, float alpha,
                        const float *A, int64_t lda, const float *B, int64_t ldb,
                        float beta, const float *C0, int64_t ldc,
                        double *R, double *D, int64_t ldr) {
    return tm_oracle_sgemm_rows(m, n, k, alpha, A, lda, B, ldb, beta, C0, ldc,
                                m, NULL, R, D, ldr);
}

/* Row partition of the distributed mode (SURVEY.md 8(b) "Partition rule";
 * generalises the paper's split(i, N/Ranks), and the rank
 * conditional q = get_rank(), to P not dividing m):
 *     rows_r = floor(m/P) + (r < m mod P),  row0_r = r*floor(m/P) + min(r, m mod P). */
int tm_oracle_dist_rows(int64_t m, int nranks, int rank, int64_t *row0, int64_t *rows) {
    if (m < 0 || nranks < 1 || rank < 0 || rank >= nranks || !row0 || !rows) return -1;
    const int64_t q = m / nranks, r = m % nranks;
    if (MUT(10)) {   /* the plausible slip: remainder rows to the last ranks */
        const int first_big = nranks - (int)r;
        *rows = q + (rank >= first_big ? 1 : 0);
        *row0 = (int64_t)rank * q + (rank > first_big ? rank - first_big : 0);
        return 0;
    }
    *rows = q + (rank < r ? 1 : 0);
    *row0 = (int64_t)rank * q + (rank < r ? rank : r);
    return 0;
}

void tm_oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int tm_oracle_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------
 * Convolution oracle ("sgemm (matrix
 * multiplication used to implement convolutions)", Conv: 512x512 input, 16
 * features, batch 32, filters 3x3..11x11).  The plain definition, fp64:
 *
 *   Y[b,y,x,f] = alpha * sum_{ky<R, kx<S, c<C} X[b, y+ky-pad, x+kx-pad, c] * Wt[f,ky,kx,c]
 *                + beta * Y0[b,y,x,f]
 *   D[b,y,x,f] = |alpha| * sum |X||Wt| + |beta| |Y0|      (acceptance denominator)
 *
 * NHWC activations, KRSC filters (F x R x S x C), stride 1, dilation 1, zero
 * padding `pad` (X outside [0,H) x [0,W) reads as 0); output Ho = H + 2 pad - R
 * + 1, Wo = W + 2 pad - S + 1.  Sum order: ky, kx, c ascending.  Special
 * cases as the GEMM oracle (beta == 0 does not read Y0; alpha == 0 does not
 * read X, Wt).  R, D are (Nb*Ho*Wo) x F row-major (ldr = F); `pixels` selects
 * output pixels (flattened b*Ho*Wo + y*Wo + x), NULL = all.
 * ---------------------------------------------------------------------- */
int tm_oracle_conv2d_nhwc(int64_t Nb, int64_t H, int64_t W, int64_t C, int64_t F, int64_t R, int64_t S,
                          int64_t pad, float alpha, const float *X, const float *Wt, float beta,
                          const float *Y0, int64_t npix, const int64_t *pixels, double *Rout, double *Dout) {
    if (Nb < 0 || H < 1 || W < 1 || C < 1 || F < 1 || R < 1 || S < 1 || pad < 0) return -1;
    const int64_t Ho = H + 2 * pad - R + 1, Wo = W + 2 * pad - S + 1;
    if (Ho < 1 || Wo < 1) return -1;
    const int64_t P = Nb * Ho * Wo;
    if (!pixels && npix != P) return -1;
    if (npix < 0 || (npix > 0 && (!Rout || !Dout))) return -1;
    if (alpha != 0.0f && (!X || !Wt)) return -1;
    if (beta != 0.0f && !Y0) return -1;
    if (pixels)
        for (int64_t t = 0; t < npix; ++t)
            if (pixels[t] < 0 || pixels[t] >= P) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < npix; ++t) {
        const int64_t q = pixels ? pixels[t] : t;
        const int64_t b = q / (Ho * Wo), y = (q / Wo) % Ho, x = q % Wo;
        for (int64_t f = 0; f < F; ++f) {
            double acc = 0.0, acc_abs = 0.0;
            if (alpha != 0.0f) {
                for (int64_t ky = 0; ky < R; ++ky) {
                    const int64_t iy = y + ky - (MUT(9) ? 0 : pad);
                    for (int64_t kx = 0; kx < S; ++kx) {
                        const int64_t ix = x + kx - pad;
                        for (int64_t c = 0; c < C; ++c) {
                            const double xv = (iy < 0 || iy >= H || ix < 0 || ix >= W)
                                                  ? 0.0 : (double)X[((b * H + iy) * W + ix) * C + c];
                            const int64_t wy = MUT(8) ? R - 1 - ky : ky, wx = MUT(8) ? S - 1 - kx : kx;
                            const double wv = (double)Wt[((f * R + wy) * S + wx) * C + c];
                            acc += xv * wv;
                            acc_abs += fabs(xv) * fabs(wv);
                        }
                    }
                }
            }
            double r = (double)alpha * acc, d = fabs((double)alpha) * acc_abs;
            if (beta != 0.0f) {
                const double c0 = (double)Y0[q * F + f];
                r += (double)beta * c0;
                d += fabs((double)beta) * fabs(c0);
            }
            Rout[t * F + f] = r;
            Dout[t * F + f] = d;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------
 * Blur oracle (the paper's distributed example, a
 * second distributed workload).  PAPER.md:216-219 (Fig. 3, the Blur algorithm):
 *
 *   bx(i,j,c) = (in(i,j,c) + in(i,j+1,c) + in(i,j+2,c)) / 3
 *   by(i,j,c) = (bx(i,j,c) + bx(i+1,j,c) + bx(i+2,j,c)) / 3
 *   0 <= i < N-2, 0 <= j < M-2, 0 <= c < 3
 *
 * written out in fp64 (the paper's element type is not stated; inputs are
 * fp32).  `in` is N x M x 3 row-major (channels interleaved, in(i,j,c) at
 * in[(i*M + j)*3 + c]); R (and the tolerance scale D = (1/9) sum of the nine
 * |in| taps) are (N-2) x (M-2) x 3.  Rows `rows[0..nrows)` of the output only
 * (NULL: all N-2).  Returns -1 on invalid arguments (N < 3 or M < 3). */
int tm_oracle_blur(int64_t N, int64_t M, const float *in, int64_t nrows, const int64_t *rows,
                   double *R, double *D) {
    if (N < 3 || M < 3 || !in || nrows < 0 || (nrows > 0 && (!R || !D))) return -1;
    if (!rows && nrows != N - 2) return -1;
    if (rows)
        for (int64_t t = 0; t < nrows; ++t)
            if (rows[t] < 0 || rows[t] >= N - 2) return -1;
    const int64_t W = M - 2;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nrows; ++t) {
        const int64_t i = rows ? rows[t] : t;
        for (int64_t j = 0; j < W; ++j) {
            for (int64_t c = 0; c < 3; ++c) {
                double bx[3], ax[3];
                for (int64_t di = 0; di < 3; ++di) {           /* bx(i+di, j, c) */
                    const float *row = in + ((i + di) * M) * 3;
                    const double a = row[j * 3 + c], b = row[(j + 1) * 3 + c];
                    const double e = row[(j + (MUT(12) ? 1 : 2)) * 3 + c];
                    bx[di] = (a + b + e) / 3.0;
                    ax[di] = (fabs(a) + fabs(b) + fabs(e)) / 3.0;
                }
                const double s = bx[0] + bx[1] + bx[2];
                R[(t * W + j) * 3 + c] = MUT(13) ? s : s / 3.0;
                D[(t * W + j) * 3 + c] = (ax[0] + ax[1] + ax[2]) / 3.0;
            }
        }
    }
    return 0;
}
