/*
 * tm.h -- C ABI of the B200-native fp32 GEMM library (libtm.so).
 *
 * The operation (SI "Introduction"): generalized matrix
 * multiplication
 *
 *     C = alpha * A * B + beta * C            (sgemm, fp32)
 *
 * in row-major storage with no transposes (reading 1, 2):
 *
 *     C[i*ldc + j] = alpha * sum_{p<k} A[i*lda + p] * B[p*ldb + j] + beta * C[i*ldc + j]
 *     for 0 <= i < m, 0 <= j < n.
 *
 * A column-major caller computes the same product by swapping operands:
 * column-major C(m x n) = A B  <=>  row-major C^T(n x m) = B^T A^T.
 *
 * Accuracy contract (BASELINE.json north_star): every element satisfies
 *     |C - C_ref| / (|alpha| * sum_p |A[i,p]||B[p,j]| + |beta||C0[i,j]|) <= 1e-5
 * against the exact result C_ref, on every path below.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - All functions are extern "C", never throw, and return tm_status.
 * - Pointers A, B, C, A_local, ... are DEVICE pointers (cudaMalloc or torch
 *   allocations on the current device) unless the name says _host.  The caller
 *   owns every buffer; the library never frees or retains caller memory.
 *   tm_sgemm / tm_sgemm_ex allocate no device memory.
 * - stream is a cudaStream_t (passed as void* so this header needs no CUDA
 *   include); NULL means the legacy default stream.  Calls are stream-ordered
 *   and return after enqueueing; device faults surface at the caller's next
 *   synchronisation on that stream.
 * - Special cases (reference-BLAS semantics, reading 5):
 *     m == 0 or n == 0        -> no-op, TM_OK;
 *     alpha == 0 or k == 0    -> A, B are not read, C = beta*C;
 *     beta == 0               -> C is not read before being written
 *                                (NaN/Inf already in C do not propagate).
 * - Invalid arguments (negative sizes, lda < max(1,k), ldb < max(1,n),
 *   ldc < max(1,n), NULL where a matrix must be read or written, C overlapping
 *   A or B) return TM_ERR_INVALID_VALUE with C untouched.
 * - A device other than sm_100 (B200) returns TM_ERR_UNSUPPORTED_DEVICE.
 *   There is no CPU fallback anywhere in this library.
 * - Determinism: for fixed inputs, algorithm and device, results are bitwise
 *   reproducible run to run (no atomics in any reduction).
 * - Thread safety: calls are reentrant; a tm_comm_t must not be used by two
 *   host threads at once (NCCL rule).
 */
#ifndef TM_H_
#define TM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TM_OK = 0,
    TM_ERR_INVALID_VALUE = 1,
    TM_ERR_UNSUPPORTED_DEVICE = 2,
    TM_ERR_CUDA = 3,
    TM_ERR_NCCL = 4,
    TM_ERR_OUT_OF_MEMORY = 5,
    TM_ERR_INTERNAL = 6
} tm_status;

/* Path selection for tm_sgemm_ex.
 *  TM_ALGO_AUTO      problems of at most 2^22 multiply-adds (m*n*k) with
 *                    k <= 256 take the small-GEMM kernel (FP32 FFMA, one CTA
 *                    per 32x32 / 64x64 tile, launch-latency bound --
 *                    BASELINE.json configs[0]);
 *                    otherwise the 3xTF32 tensor-core path when its layout
 *                    rules hold (A, B, C 16-byte aligned; lda, ldb, ldc
 *                    multiples of 4), else the SIMT path.  Misalignment is
 *                    never an error here.
 *  TM_ALGO_TF32X3    3xTF32 split-operand tcgen05 MMA (fp32 result, TMEM
 *                    accumulation).  Misaligned input -> TM_ERR_INVALID_VALUE.
 *  TM_ALGO_SIMT_F32  pure-FP32 FFMA register-blocked kernel (validation path).
 *  TM_ALGO_TF32X1    single-pass TF32 precision variant:
 *                    one tcgen05 kind::tf32 MMA per K step on the raw fp32
 *                    operands, which the tensor core truncates to TF32 (10
 *                    explicit mantissa bits).  Per product |a_hi b_hi - ab| <=
 *                    2^-9 |a||b|; with the accumulation of the 3xTF32 path
 *                    (round-toward-zero partials of K_c = 128, RN promotion)
 *                    max |C - R| / D <= 2^-9 + 2^-14 for k <= 4096 -- about
 *                    2e-3; it does NOT meet the 1e-5 contract and AUTO never
 *                    selects it.  Integer inputs |x| <= 2048 are exact in TF32,
 *                    so their products are exact.  Same layout rules,
 *                    transposes and special cases as TF32X3.
 *  TM_ALGO_BF16X9    BF16x9 precision variant: every
 *                    fp32 operand is split in the kernel into three bf16
 *                    pieces x = b0 + b1 + b2 (b0 = RN_bf16(x), b1 =
 *                    RN_bf16(x - b0), b2 = x - b0 - b1; exact for normal fp32:
 *                    8 + 8 + 8 significant bits) and all nine products a_i b_j
 *                    run on kind::f16 tcgen05 MMAs -- each product exact in
 *                    fp32, so the only error is the fp32 accumulation (the
 *                    3xTF32 path's scheme: round-toward-zero partials of K_c =
 *                    128, RN promotion), about 1.5x as many roundings per K as
 *                    TF32X3 and no representation error (TF32X3: 2^-19 per
 *                    product).  Meets the 1e-5 contract (tests/test_bf16x9.py);
 *                    integer inputs are bit-exact.  Runs at the bf16 tensor
 *                    rate / 9 (TF32X3: tf32 rate / 3, about 1.5x faster), so
 *                    AUTO never selects it.  Same layout rules, transposes and
 *                    special cases as TF32X3. */
typedef enum {
    TM_ALGO_AUTO = 0,
    TM_ALGO_TF32X3 = 1,
    TM_ALGO_SIMT_F32 = 2,
    TM_ALGO_TF32X1 = 3,
    TM_ALGO_BF16X9 = 4
} tm_algo;

/* C = alpha*A*B + beta*C on `stream`.  A: m x k (lda),
 * B: k x n (ldb), C: m x n (ldc), all row-major fp32 device memory.
 * CUDA graphs: the call enqueues only kernels and memsets, so it may be
 * captured (stream capture) and replayed.  Stream-K schedules use a small
 * library workspace per (device, stream) that cannot be allocated during
 * capture: make the same call once on the capturing stream before capturing
 * (otherwise TM_ERR_INVALID_VALUE); replay on that stream (or serialised with
 * it).  Workspaces are never freed while the process runs, so captured graphs
 * stay valid. */
tm_status tm_sgemm(int64_t m, int64_t n, int64_t k, float alpha,
                   const float* A, int64_t lda, const float* B, int64_t ldb,
                   float beta, float* C, int64_t ldc, void* stream);

/* Same operation with an explicit path (tm_algo). */
tm_status tm_sgemm_ex(int64_t m, int64_t n, int64_t k, float alpha,
                      const float* A, int64_t lda, const float* B, int64_t ldb,
                      float beta, float* C, int64_t ldc, void* stream, int algo);

/* Transposed operands (BLAS op(); SURVEY.md 8(f) item 1 -- the paper's gemm,
 * PAPER.md:67, has none).  Row-major storage throughout:
 *   opa == TM_OP_N: A is m x k (lda >= max(1,k)), op(A)[i,p] = A[i*lda + p]
 *   opa == TM_OP_T: A is k x m (lda >= max(1,m)), op(A)[i,p] = A[p*lda + i]
 *   opb == TM_OP_N: B is k x n (ldb >= max(1,n)), op(B)[p,j] = B[p*ldb + j]
 *   opb == TM_OP_T: B is n x k (ldb >= max(1,k)), op(B)[p,j] = B[j*ldb + p]
 * C = alpha*op(A)*op(B) + beta*C, C m x n (ldc).  Same paths, accuracy, special
 * cases and errors as tm_sgemm_ex. */
typedef enum { TM_OP_N = 0, TM_OP_T = 1 } tm_op;
tm_status tm_sgemm_op(int opa, int opb, int64_t m, int64_t n, int64_t k, float alpha,
                      const float* A, int64_t lda, const float* B, int64_t ldb,
                      float beta, float* C, int64_t ldc, void* stream, int algo);

/* Reference-BLAS (column-major) sgemm: C = alpha*op(A)*op(B) + beta*C with
 * transa/transb in {'N','T','C'} ('C' == 'T' for real data), A, B, C
 * column-major with leading dimensions lda, ldb, ldc as in BLAS.  Implemented
 * as the row-major product C^T = op(B)^T op(A)^T (no data movement). */
tm_status tm_sgemm_colmajor(char transa, char transb, int64_t m, int64_t n, int64_t k, float alpha,
                            const float* A, int64_t lda, const float* B, int64_t ldb,
                            float beta, float* C, int64_t ldc, void* stream);

/* 2-D convolution as a GEMM (the paper's Conv
 * benchmark, "sgemm ... used to implement convolutions"):
 * stride 1, dilation 1,
 * zero padding `pad`, device pointers
 *   X  : nb x h x w x c        (NHWC, dense)
 *   Wt : f x r x s x c         (KRSC filters, dense)
 *   Y  : nb x ho x wo x f      (NHWC, dense), ho = h + 2 pad - r + 1, wo = w + 2 pad - s + 1
 *   Y[b,y,x,f] = alpha * sum_{ky,kx,c} X[b, y+ky-pad, x+kx-pad, c] * Wt[f,ky,kx,c] + beta * Y[b,y,x,f]
 * (X outside the image reads as zero).  AUTO uses a 3xTF32 tensor-core path
 * when c % 16 == 0, f % 4 == 0, pointers 16-byte aligned and pad <= 127 --
 * the direct halo-tile kernel when s <= 24, c <= 128 and f <= 64 (the
 * reduction over filter rows runs in passes; filters whose resident hi + lo
 * copies exceed shared memory, e.g. 11x11 x 16 channels, are split over two
 * launches by filter column, the second accumulating with beta = 1; see
 * tm_conv2d_plan_name), else the implicit-GEMM kernel (A =
 * im2col of X streamed by TMA im2col-mode copies, never materialised) -- and
 * otherwise the FP32 SIMT direct convolution; TM_ALGO_TF32X3 on shapes
 * outside the tensor-core rule returns TM_ERR_INVALID_VALUE.  Same accuracy contract (normalised by
 * |alpha| sum |X||Wt| + |beta||Y|), special cases and errors as tm_sgemm_ex. */
tm_status tm_conv2d_nhwc(int64_t nb, int64_t h, int64_t w, int64_t c, int64_t f, int64_t r, int64_t s,
                         int64_t pad, float alpha, const float* X, const float* Wt, float beta, float* Y,
                         void* stream, int algo);

/* Name of the kernel tm_conv2d_nhwc would run for these arguments ("direct",
 * "direct_split" -- the direct kernel in two launches over the filter
 * columns -- "implicit_gemm", "simt", "scale", "noop" or "invalid"); host-only, no
 * launch (pointers are only inspected for alignment). */
const char* tm_conv2d_plan_name(int64_t nb, int64_t h, int64_t w, int64_t c, int64_t f, int64_t r, int64_t s,
                                int64_t pad, float alpha, const float* X, const float* Wt, const float* Y, int algo);

/* End-to-end entry with HOST buffers (ideally pinned): copies A, B (and C when
 * beta != 0) to the current device, computes, copies C back, and synchronises
 * `stream` before returning.  Host->device copies of row blocks of A/C overlap
 * the GEMM of the previous block.  Device staging memory is owned by the
 * library (grown on demand, cached per device; released by tm_release_workspace).
 * Errors as above; TM_ERR_OUT_OF_MEMORY if staging cannot be allocated. */
tm_status tm_sgemm_host(int64_t m, int64_t n, int64_t k, float alpha,
                        const float* A_host, int64_t lda, const float* B_host, int64_t ldb,
                        float beta, float* C_host, int64_t ldc, void* stream, int algo);

/* Frees the staging buffers tm_sgemm_host cached on the current device. */
tm_status tm_release_workspace(void);

/* Human-readable name of a status code (static storage, never NULL). */
const char* tm_status_string(tm_status s);

/* Library version as major*10000 + minor*100 + patch. */
int tm_get_version(void);

/* Measured configuration choice (the paper auto-tuned
 * its sgemm's tile sizes).  Times every compiled 3xTF32
 * tensor-core configuration -- 1- or 2-SM CTA group x 32/64/128-column CTA
 * tile x data-parallel/stream-K schedule -- on these operands (op(A), op(B) as
 * in tm_sgemm_op; `reps` timed runs each after one warm-up, median kept) and
 * records the fastest in a process-wide cache keyed by (m, n, k, opa, opb,
 * beta != 0, SM count); later AUTO/TF32X3 calls with that key use it.  The
 * trials write a library-allocated scratch copy of C: the caller's C is only
 * read (when beta != 0) and is unchanged.  Device pointers, stream-ordered
 * but synchronising (it reads the timings).  Outputs (may be NULL): the chosen
 * cg (1/2), bn_cta (32/64/128), streamk (0/1) and its median time in ms.
 * Errors: TM_ERR_INVALID_VALUE if tm_sgemm_op(..., TM_ALGO_TF32X3) would reject
 * the arguments, if m, n or k is 0, alpha == 0 or reps is outside [1, 1000];
 * TM_ERR_CUDA on allocation or launch failure. */
tm_status tm_sgemm_tune(int opa, int opb, int64_t m, int64_t n, int64_t k, float alpha, const float* A, int64_t lda,
                        const float* B, int64_t ldb, float beta, const float* C, int64_t ldc, void* stream, int reps,
                        int* best_cg, int* best_bn, int* best_streamk, float* best_ms);

/* Tuning cache management (host-only).  File format: one entry per line,
 * "m n k opa opb beta_nonzero sms cg bn_cta streamk" ('#' lines are comments);
 * load skips malformed entries and returns how many it added (-1 if the file
 * cannot be opened); save overwrites `path`. */
int tm_tune_cache_size(void);
tm_status tm_tune_cache_clear(void);
tm_status tm_tune_cache_save(const char* path);
int tm_tune_cache_load(const char* path);

/* The plan tm_sgemm_op(opa, opb, ..., algo) would use (host-only, no launch):
 * *path = 0 invalid, 1 no-op, 2 scale, 3 tensor cores, 4 SIMT, 5 small-GEMM
 * SIMT kernel; for tensor
 * cores the CTA group, CTA tile width and schedule (tuned entry if cached,
 * else the cost model).  Output pointers may be NULL.  Returns
 * TM_ERR_INVALID_VALUE for arguments the call would reject. */
tm_status tm_sgemm_plan_config(int opa, int opb, int64_t m, int64_t n, int64_t k, float alpha, const float* A,
                               int64_t lda, const float* B, int64_t ldb, float beta, const float* C, int64_t ldc,
                               int algo, int* path, int* cg, int* bn_cta, int* streamk);

/* Stream-K work split of a tensor-core launch (host-only, no device): of
 * `num_tiles` output tiles of `kblocks` K-blocks (32 k each) on `clusters`
 * persistent clusters, *sk_tiles tiles (the first in the grouped raster) are
 * cut into equal contiguous ranges of tile x K-block iterations, one per
 * cluster, and reduced in cluster order; the remaining tiles run whole,
 * data-parallel, after each cluster's share (the "hybrid" schedule;
 * *sk_tiles == num_tiles is pure stream-K).  *clusters_used is the launch's
 * cluster count (fewer than `clusters` only when there are fewer than two
 * iterations per cluster).  mode: 0 pure stream-K, 1 the partial wave's
 * tiles, 2 those plus one full wave, -1 the library default (2 when
 * kblocks < 64, else 1).  Guarantees: every cluster owns >= 2 iterations of
 * the region; num_tiles - *sk_tiles is a multiple of *clusters_used.  The
 * paper's tiled loop nest (PAPER.md:753-758 tiling, 830-831 the GPU gemm)
 * fixes the result of each tile, not this split.  TM_ERR_INVALID_VALUE on
 * num_tiles, kblocks or clusters < 1, mode > 2, or null outputs. */
tm_status tm_sgemm_streamk_region(int64_t num_tiles, int64_t kblocks, int clusters, int mode, int64_t* sk_tiles,
                                  int* clusters_used);

/* Name of the path tm_sgemm_ex would take for these arguments on the current
 * device ("tf32x3", "tf32x1", "simt", "simt_small", "scale", "noop", or
 * "invalid"); host-only, no launch. */
const char* tm_sgemm_plan_name(int64_t m, int64_t n, int64_t k, float alpha,
                               const float* A, int64_t lda, const float* B, int64_t ldb,
                               float beta, const float* C, int64_t ldc, int algo);

/* ---------------------------------------------------------------------------
 * Multi-GPU row-sharded mode (one process per GPU).
 *
 * Follows the paper's distribution model: data is distributed across ranks by
 * rows, each rank computes its own row block
 * (distribute(i); rank conditional q = get_rank(),
 * PAPER.md:784-794) and no gather of C is performed.
 * The only exchange is B: broadcast from `root` (or all-gathered from k-row
 * shards) with NCCL over NVLink, in K-chunks that overlap the GEMM of the
 * previous chunk.
 * ------------------------------------------------------------------------- */
typedef struct tm_comm_s* tm_comm_t;
typedef struct { unsigned char bytes[128]; } tm_unique_id; /* wraps ncclUniqueId */

/* Rank 0 creates the id and ships it to all ranks (e.g. torch.distributed). */
tm_status tm_comm_get_unique_id(tm_unique_id* out);

/* Collective over `nranks` processes; binds to the CURRENT CUDA device.  The
 * communicator owns one comm stream and its chunk events. */
tm_status tm_comm_init(tm_comm_t* out, int nranks, int rank, const tm_unique_id* id);
tm_status tm_comm_destroy(tm_comm_t comm);
tm_status tm_comm_rank(tm_comm_t comm, int* rank, int* nranks);

/* Balanced block partition of m rows over nranks:
 *   rows = m/P + (rank < m%P),  row0 = rank*(m/P) + min(rank, m%P). */
tm_status tm_dist_rows(int64_t m, int nranks, int rank, int64_t* row0, int64_t* rows);

/* K-chunk schedule of tm_sgemm_dist (host-only, no device): number of chunks
 * B is broadcast in for this (k, nranks), and chunk `idx`'s K range
 * [*k0, *k0 + *kr).  Chunks tile [0, k) exactly once, in order; every chunk
 * but the last starts at a multiple of 32.  idx < 0 only returns the count
 * in *k0. */
tm_status tm_dist_chunk(int64_t k, int nranks, int idx, int64_t* k0, int64_t* kr);

/* Collective: all ranks call with identical m, n, k, alpha, beta, root.
 *   A_local: rows x k (lda), C_local: rows x n (ldc), rows from tm_dist_rows.
 *   B: k x n (ldb); valid on `root`; on other ranks a caller-owned k*ldb
 *      device buffer that is overwritten with root's B.  Whole rows of ldb
 *      floats are transferred, so on EVERY rank B must be a buffer of k*ldb
 *      floats (the root's last row is read up to k*ldb, past the last valid
 *      element (k-1)*ldb + n), and on receivers the padding columns [n, ldb)
 *      of each row are overwritten too: a column-slice view of a wider matrix
 *      would have its neighbouring columns clobbered -- pass ldb == n then.
 * On return (stream-ordered) C_local = alpha*A_local*B + beta*C_local. */
tm_status tm_sgemm_dist(tm_comm_t comm, int64_t m, int64_t n, int64_t k, float alpha,
                        const float* A_local, int64_t lda, float* B, int64_t ldb, int root,
                        float beta, float* C_local, int64_t ldc, void* stream);

/* Fused single-launch variant of tm_sgemm_dist (same arguments and result;
 * SURVEY.md 8(e) "Fused alternative"): ONE persistent tensor-core GEMM over
 * the full K runs while B's K-chunks are broadcast; after each chunk the comm
 * stream sets a device flag with a stream memory operation
 * (cuStreamWriteValue32) and the GEMM's TMA producers wait for chunk c's flag
 * before loading any stage of it.  No beta chain (C read and written once)
 * and one launch tail instead of one per chunk.  The GEMM leaves SMs free for
 * the NCCL kernels.  Falls back to the chunked schedule when the operands do
 * not meet the tensor-core layout rules.  A transfer that never completes
 * makes the GEMM trap after ~20 s (TM_ERR_CUDA at the next synchronisation)
 * instead of hanging the device. */
tm_status tm_sgemm_dist_fused(tm_comm_t comm, int64_t m, int64_t n, int64_t k, float alpha,
                              const float* A_local, int64_t lda, float* B, int64_t ldb, int root,
                              float beta, float* C_local, int64_t ldc, void* stream);

/* Single-process loopback of the distributed mode (verification, DESIGN.md
 * section 10): emulates `nranks` ranks one after another on the CURRENT device
 * with the identical partition, schedule and beta chain as the NCCL entry
 * points; every transfer is a device-to-device copy.
 *   mode 0: tm_sgemm_dist -- Bs[root] holds B, the other Bs[r] are overwritten
 *           chunk by chunk ("broadcast").
 *   mode 1: tm_sgemm_dist_allgather -- Bs[r] holds rank r's k-row shard at rows
 *           [r*k/P, (r+1)*k/P) (k % nranks == 0); every Bs[r] ends complete.
 *   mode 2: tm_sgemm_dist_fused -- as mode 0, with one flag-gated GEMM per
 *           rank; the chunk copies and the flag writes run on a separate
 *           stream concurrently with it.
 *   mode 3, 4: modes 0 and 2 under the copy-engine transport model
 *           (tm_sgemm_dist_ce between devices: peer copies run on the copy
 *           engines, which one device cannot emulate -- its own device-to-
 *           device copies are kernels): NO data moves, the caller fills every
 *           Bs[r] with B beforehand; chunk c is only released on the link
 *           model's schedule (rate TM_LOOPBACK_LINK_GBS, default 700 GB/s) and
 *           the GEMMs keep every SM but one (the pacing kernel's).  Timing
 *           projections; the result is still checked by the tests.
 *   Env TM_LOOPBACK_LINK_GBS = R (projections): chunk c of the rank at chain
 *   position q (root 0) is released no earlier than (q * 128 K-rows + bytes
 *   of chunks 0..c) / R after the rank's transfers start, modelling a
 *   pipelined chain (or ring) of links of rate R; in modes 0-2 also no
 *   earlier than its device copy completes.
 *   A_locals[r], Bs[r], C_locals[r]: device pointers (host arrays of nranks),
 *   shaped as the NCCL entry's A_local, B / B_full, C_local for rank r.
 *   bytes_received: optional host array of nranks counters (bytes each rank's
 *   B received), or NULL.
 * Synchronises `stream`; errors as tm_sgemm_dist. */
tm_status tm_sgemm_dist_loopback(int nranks, int root, int mode, int64_t m, int64_t n, int64_t k, float alpha,
                                 const float* const* A_locals, int64_t lda, float* const* Bs, int64_t ldb,
                                 float beta, float* const* C_locals, int64_t ldc, uint64_t* bytes_received,
                                 void* stream);

/* Variant: B is pre-sharded by k-rows (B_shard = rows [k0, k0+kr) of B from
 * tm_dist_rows(k, ...), leading dimension ldb), all-gathered into the
 * caller-owned B_full (k x n, ldb).  Requires every rank's shard to have the
 * same row count (k % nranks == 0), as ncclAllGather does.  Buffer extents:
 * whole rows of ldb floats move, so B_shard must be kr*ldb floats and B_full
 * k*ldb floats (kr = k/nranks), and the padding columns [n, ldb) of B_full are
 * overwritten with the shards' padding -- pass ldb == n for column-slice views. */
tm_status tm_sgemm_dist_allgather(tm_comm_t comm, int64_t m, int64_t n, int64_t k, float alpha,
                                  const float* A_local, int64_t lda, const float* B_shard,
                                  float* B_full, int64_t ldb, float beta, float* C_local,
                                  int64_t ldc, void* stream);

/* ---------------------------------------------------------------------------
 * 2-D SUMMA sharding ("2-D SUMMA-style sharding for
 * larger P"; the paper's distribute / send / receive, PAPER.md:311,
 * PAPER.md:323-335, generalised from rows to a grid).
 *
 * nranks = pr * pc; rank r is grid position (i, j) = (r / pc, r % pc) and owns
 *   C_local = C[rows_i, cols_j]   (rows_i x cols_j, ldc)
 *   A_local = A[rows_i, ka_j]     (rows_i x |ka_j|, lda >= |ka_j|)
 *   B_local = B[kb_i, cols_j]     (|kb_i| x cols_j, ldb >= cols_j)
 * with rows_i = tm_dist_rows(m, pr, i), cols_j = tm_dist_rows(n, pc, j),
 * ka_j = tm_dist_rows(k, pc, j), kb_i = tm_dist_rows(k, pr, i).  K is cut into
 * panels (tm_summa_panel) each inside one A column block and one B row block;
 * per panel the owner of A(i, panel) broadcasts it along grid row i and the
 * owner of B(panel, j) along grid column j (NCCL, row / column communicators
 * split from the communicator on the first call with a grid), and every rank
 * accumulates C_local = alpha * A(i, panel) B(panel, j) + beta_p C_local (beta
 * for the first panel, then 1).  Panels are double-buffered in library memory
 * owned by the communicator.  On return (stream-ordered) C_local = alpha *
 * A[rows_i, :] B[:, cols_j] + beta C_local; inputs are not modified.
 * Collective: all ranks call with the same pr, pc, m, n, k, alpha, beta.
 * Errors: pr * pc != nranks or bad sizes -> TM_ERR_INVALID_VALUE; NCCL
 * failure -> TM_ERR_NCCL; panel buffers -> TM_ERR_OUT_OF_MEMORY. */
tm_status tm_sgemm_summa(tm_comm_t comm, int pr, int pc, int64_t m, int64_t n, int64_t k, float alpha,
                         const float* A_local, int64_t lda, const float* B_local, int64_t ldb, float beta,
                         float* C_local, int64_t ldc, void* stream);

/* Panel plan of tm_sgemm_summa (host-only): idx < 0 returns the panel count in
 * *k0; otherwise panel idx's K range [*k0, *k0 + *kr).  Panels tile [0, k) in
 * order, each inside one block of tm_dist_rows(k, pc, .) and of
 * tm_dist_rows(k, pr, .), at most 2048 long. */
tm_status tm_summa_panel(int64_t k, int pr, int pc, int idx, int64_t* k0, int64_t* kr);

/* Single-process loopback of tm_sgemm_summa (verification): pr * pc simulated
 * ranks on the current device one after another; every panel is packed
 * straight from its owner's block (device copies) instead of broadcast.
 * Arrays of nranks entries: A_locals / ldas, B_locals / ldbs, C_locals / ldcs
 * as rank r's arguments; bytes_received: optional per-rank counters of panel
 * bytes that came from another rank.  Synchronises `stream`. */
tm_status tm_sgemm_summa_loopback(int pr, int pc, int64_t m, int64_t n, int64_t k, float alpha,
                                  const float* const* A_locals, const int64_t* ldas, const float* const* B_locals,
                                  const int64_t* ldbs, float beta, float* const* C_locals, const int64_t* ldcs,
                                  uint64_t* bytes_received, void* stream);

/* ---------------------------------------------------------------------------
 * Copy-engine chain broadcast (the paper's explicit
 * send/receive between row-owning ranks).
 *
 * Same result as tm_sgemm_dist, but B travels root -> root+1 -> ... as a
 * pipelined chain of device-to-device copies into the successor's buffer
 * through CUDA IPC mappings -- executed by the copy engines, so the GEMM keeps
 * every SM (tm_sgemm_dist leaves 16 to NCCL's kernels).  Each 128-K-row piece
 * is flagged on arrival with a stream memory operation; a rank gives its
 * predecessor a credit (its B is free) at the start of every call.
 *
 * Bootstrap (no NCCL): every rank calls tm_ce_create, all-gathers the
 * exported flag handles (any host transport, e.g. torch.distributed), then
 * tm_ce_connect.  Every call passes the all-gathered tm_ipc_export of each
 * rank's B buffer (re-export when a buffer changes).  Device memory must come
 * from cudaMalloc (or torch's default caching allocator); one process per
 * device, or several processes sharing a device (the tests do).  A tm_ce_t
 * must not be used by two host threads at once; peer mappings it opened stay
 * mapped until tm_ce_destroy.
 * ------------------------------------------------------------------------- */
typedef struct { unsigned char bytes[64]; int64_t offset; } tm_ipc_buf; /* IPC handle of the allocation + byte offset */
typedef struct tm_ce_s* tm_ce_t;

/* Exports the allocation containing the device pointer `ptr` (cudaIpcGetMemHandle
 * of its base) and ptr's offset in it.  TM_ERR_INVALID_VALUE if ptr is not
 * device memory of this process, TM_ERR_CUDA if the allocation cannot be
 * exported (e.g. virtual-memory-API allocations). */
tm_status tm_ipc_export(const void* ptr, tm_ipc_buf* out);

/* Creates this rank's chain endpoint on the CURRENT device (its flag array,
 * two streams, events) and exports the flags in *my_flags. */
tm_status tm_ce_create(tm_ce_t* out, int nranks, int rank, tm_ipc_buf* my_flags);
/* Maps every peer's flags (all_flags: nranks entries, all-gathered from
 * tm_ce_create).  Collective in the sense that all ranks must call it before
 * the first tm_sgemm_dist_ce. */
tm_status tm_ce_connect(tm_ce_t ce, const tm_ipc_buf* all_flags);
/* Synchronises the endpoint's streams, unmaps peers and frees it. */
tm_status tm_ce_destroy(tm_ce_t ce);
/* Bytes of B this rank received through the chain since tm_ce_create. */
tm_status tm_ce_bytes_received(tm_ce_t ce, uint64_t* bytes);

/* Collective: all ranks call with identical m, n, k, alpha, beta, root, fused,
 * in the same order.  Arguments as tm_sgemm_dist (B: a k*ldb device buffer on
 * every rank, valid on root, overwritten elsewhere; whole rows move), plus
 * all_B: nranks tm_ipc_export records of every rank's B.  fused != 0: one
 * flag-gated GEMM over the full K (tm_sgemm_dist_fused's kernel, gated per
 * piece); 0: the K-chunked schedule with every SM.  Stream-ordered; on return
 * (stream-ordered) C_local = alpha*A_local*B + beta*C_local and B is complete.
 * A peer that never makes its call leaves this rank's streams waiting (no
 * timeout in the copy chain; the fused GEMM traps after ~20 s). */
tm_status tm_sgemm_dist_ce(tm_ce_t ce, int64_t m, int64_t n, int64_t k, float alpha,
                           const float* A_local, int64_t lda, float* B, int64_t ldb,
                           const tm_ipc_buf* all_B, int root, float beta, float* C_local,
                           int64_t ldc, int fused, void* stream);

/* ---------------------------------------------------------------------------
 * Blur: the paper's second distributed workload.
 *
 * The two-stage 3x3 box blur of PAPER.md:216-219 (Fig. 3):
 *     bx(i,j,c) = (in(i,j,c) + in(i,j+1,c) + in(i,j+2,c)) / 3
 *     by(i,j,c) = (bx(i,j,c) + bx(i+1,j,c) + bx(i+2,j,c)) / 3
 *     for 0 <= i < N-2, 0 <= j < M-2, 0 <= c < 3
 * (the paper ignores boundary conditions, so the output is (N-2) x (M-2) x 3).
 * Layout (the paper's in[i][j][c], channels interleaved): row i of the image
 * is 3M floats at in + i*ldi, in(i,j,c) = in[i*ldi + 3j + c], ldi >= 3M; row i
 * of the output is 3(M-2) floats at out + i*ldo, ldo >= 3(M-2).  Device
 * pointers; `in` spans (N-1)*ldi + 3M floats, `out` (N-3)*ldo + 3(M-2).
 * Arithmetic: fp32, "/ 3" as a multiply by fl(1/3); |by - exact| <= 1e-6 * D
 * with D = (1/9) sum of the nine |in| taps (blur accuracy).
 * Deterministic.  Vector loads/stores are used when in/out are 16-byte aligned
 * and ldi/ldo multiples of 4 (8-byte / even for 2-wide stores); any alignment
 * is accepted.
 * Errors: N < 3, M < 3, NULL pointers, ldi < 3M, ldo < 3(M-2) or out
 * overlapping in -> TM_ERR_INVALID_VALUE (out untouched). */
tm_status tm_blur(int64_t N, int64_t M, const float* in, int64_t ldi, float* out, int64_t ldo, void* stream);

/* Row-distributed blur (Fig. 5 Code 3; collective over the
 * communicator).  The N-2 output rows are partitioned with tm_dist_rows(N-2,
 * P, r): rank r computes output rows [row0, row0 + rows).  Its local image
 * `lin` holds rows + 2 rows of pitch ldi: rows [0, rows) are input rows
 * [row0, row0 + rows) (the rank's chunk); rows [rows,
 * rows + 2) are the border region: on the last rank the caller fills them
 * with input rows N-2 and N-1, on every other rank they are OVERWRITTEN with
 * the first two rows of rank r+1's chunk, received over NCCL (the paper's
 * send from node is to is-1 / receive at lin(N,0,0) from ir+1, PAPER.md:
 * 581-582: 2 rows, here ldi + 3M floats).  `lout`: rows x 3(M-2) (pitch ldo).
 * The interior output rows [0, rows - 2) are computed while the border rows
 * are in flight; the last two once they have arrived.  No gather of the
 * output.  Requires (N-2)/P >= 2 when P > 1 (every chunk
 * holds the two rows its upper neighbour needs), else TM_ERR_INVALID_VALUE.
 * Stream-ordered; errors as tm_blur, TM_ERR_NCCL on communication failure. */
tm_status tm_blur_dist(tm_comm_t comm, int64_t N, int64_t M, float* lin, int64_t ldi, float* lout, int64_t ldo,
                       void* stream);

/* Single-process loopback of tm_blur_dist (verification): `nranks` simulated
 * ranks on the current device, lins[r] / louts[r] as rank r's lin / lout;
 * the border-row exchange is a device-to-device copy on a separate stream,
 * with the identical schedule.  bytes_received: optional host array of nranks
 * counters.  Synchronises `stream`. */
tm_status tm_blur_dist_loopback(int nranks, int64_t N, int64_t M, float* const* lins, int64_t ldi,
                                float* const* louts, int64_t ldo, uint64_t* bytes_received, void* stream);

/* Failure detection: polls the communicator for asynchronous NCCL errors
 * (e.g. a peer died or a network/NVLink fault).  TM_OK if healthy (or an
 * operation is still in progress), TM_ERR_NCCL if an error was reported; with
 * abort_on_error != 0 the communicator is then aborted so that blocked
 * collectives return (tm_comm_destroy must still be called). */
tm_status tm_comm_check(tm_comm_t comm, int abort_on_error);

/* Bytes this rank received over the communicator since tm_comm_init
 * (message-conservation accounting used by the tests). */
tm_status tm_comm_bytes_received(tm_comm_t comm, uint64_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* TM_H_ */
