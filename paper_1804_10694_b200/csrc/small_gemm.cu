// small_gemm.cu -- latency-bound small sgemm, C = alpha*op(A)*op(B) + beta*C
// in plain FP32 FFMA.
//
// For problems of a few MFLOP (BASELINE.json configs[0], 64^3) the persistent
// tensor-core kernel is all fixed cost: a 512-thread cluster launch with ~200
// KB of shared memory, TMEM allocation, descriptor prefetch and an mbarrier
// pipeline that never fills (~4 us of kernel for one tile).  What bounds a
// small GEMM is the DRAM round trip of its operands and of C, so this kernel
// does only that: one CTA of 256 threads per TM x TN output tile (enough tiles
// to spread over the SMs), beta*C loaded into registers before the main loop
// so its latency hides behind the operand loads, operands staged through
// shared memory in BK = 32 slices with the next TWO slices' global loads in
// flight (registers, double-buffered: at k = 64 both slices leave in the first
// round trip instead of the second waiting for the first), and a predicated
// epilogue (full/partial
// tile separation).  Each output is the fp32 FMA chain over
// p = 0..k-1 in order (the textbook loop in fp32).
#include <cuda_runtime.h>

#include <cstdint>

#include "tm_internal.h"

namespace tmk {
namespace {

constexpr int kSmallThreads = 256;
constexpr int kSmallBK = 32;

struct SmallParams {
  const float* A;
  const float* B;
  float* C;
  int64_t lda, ldb, ldc;
  int m, n, k;
  float alpha, beta;
};

// op(A)[i, p] and op(B)[p, j] (row-major storage; TA: A stored k x m, TB: B stored n x k)
template <bool TA>
__device__ __forceinline__ float ld_a(const SmallParams& p, int i, int q) {
  return __ldg(TA ? p.A + static_cast<int64_t>(q) * p.lda + i : p.A + static_cast<int64_t>(i) * p.lda + q);
}
template <bool TB>
__device__ __forceinline__ float ld_b(const SmallParams& p, int q, int j) {
  return __ldg(TB ? p.B + static_cast<int64_t>(j) * p.ldb + q : p.B + static_cast<int64_t>(q) * p.ldb + j);
}

template <int TM, int TN, bool TA, bool TB>
__global__ void __launch_bounds__(kSmallThreads) k_sgemm_small(SmallParams p) {
  constexpr int RM = TM / 16, RN = TN / 16;        // outputs per thread (rows x cols), strided by 16
  constexpr int LA = TM * kSmallBK / kSmallThreads;  // A elements per thread per slice
  constexpr int LB = kSmallBK * TN / kSmallThreads;
  __shared__ float As[kSmallBK][TM + 1];  // k-major: As[q][i]; +1 keeps the transposing stores conflict-free
  __shared__ float Bs[kSmallBK][TN + 1];
  const int t = threadIdx.x, tx = t % 16, ty = t / 16;
  const int bm = blockIdx.y * TM, bn = blockIdx.x * TN;

  // beta*C first: its DRAM latency overlaps the operand loads below
  float cv[RM][RN];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < RN; ++c) {
      const int i = bm + ty + 16 * r, j = bn + tx + 16 * c;
      cv[r][c] = (p.beta != 0.0f && i < p.m && j < p.n) ? p.C[static_cast<int64_t>(i) * p.ldc + j] : 0.0f;
    }

  // slice element e of a thread: A (i, q) with the contiguous index fastest
  // across the warp (q for A, i for A^T), B (q, j) likewise (j for B, q for B^T)
  auto a_coord = [&](int e, int& i, int& q) {
    const int idx = e * kSmallThreads + t;
    if (TA) { i = idx % TM; q = idx / TM; } else { q = idx % kSmallBK; i = idx / kSmallBK; }
  };
  auto b_coord = [&](int e, int& q, int& j) {
    const int idx = e * kSmallThreads + t;
    if (TB) { q = idx % kSmallBK; j = idx / kSmallBK; } else { j = idx % TN; q = idx / TN; }
  };
  float ra[2][LA], rb[2][LB];
  auto fetch = [&](int k0, float (&xa)[LA], float (&xb)[LB]) {
#pragma unroll
    for (int e = 0; e < LA; ++e) {
      int i, q;
      a_coord(e, i, q);
      xa[e] = (bm + i < p.m && k0 + q < p.k) ? ld_a<TA>(p, bm + i, k0 + q) : 0.0f;
    }
#pragma unroll
    for (int e = 0; e < LB; ++e) {
      int q, j;
      b_coord(e, q, j);
      xb[e] = (k0 + q < p.k && bn + j < p.n) ? ld_b<TB>(p, k0 + q, bn + j) : 0.0f;
    }
  };
  auto stage = [&](const float (&xa)[LA], const float (&xb)[LB]) {
#pragma unroll
    for (int e = 0; e < LA; ++e) {
      int i, q;
      a_coord(e, i, q);
      As[q][i] = xa[e];
    }
#pragma unroll
    for (int e = 0; e < LB; ++e) {
      int q, j;
      b_coord(e, q, j);
      Bs[q][j] = xb[e];
    }
  };

  float acc[RM][RN];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < RN; ++c) acc[r][c] = 0.0f;

  fetch(0, ra[0], rb[0]);
  if (kSmallBK < p.k) fetch(kSmallBK, ra[1], rb[1]);
  int buf = 0;
  for (int k0 = 0; k0 < p.k; k0 += kSmallBK, buf ^= 1) {
    if (buf == 0) stage(ra[0], rb[0]);
    else stage(ra[1], rb[1]);
    __syncthreads();
    if (k0 + 2 * kSmallBK < p.k) {  // the slice after next, in flight during the FMAs
      if (buf == 0) fetch(k0 + 2 * kSmallBK, ra[0], rb[0]);
      else fetch(k0 + 2 * kSmallBK, ra[1], rb[1]);
    }
    const int kk = p.k - k0 < kSmallBK ? p.k - k0 : kSmallBK;
    for (int q = 0; q < kk; ++q) {
      float a[RM], b[RN];
#pragma unroll
      for (int r = 0; r < RM; ++r) a[r] = As[q][ty + 16 * r];
#pragma unroll
      for (int c = 0; c < RN; ++c) b[c] = Bs[q][tx + 16 * c];
#pragma unroll
      for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < RN; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);  // p ascending
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < RN; ++c) {
      const int i = bm + ty + 16 * r, j = bn + tx + 16 * c;
      if (i < p.m && j < p.n)
        p.C[static_cast<int64_t>(i) * p.ldc + j] =
            p.beta == 0.0f ? p.alpha * acc[r][c] : fmaf(p.alpha, acc[r][c], p.beta * cv[r][c]);
    }
}

template <int TM, int TN>
void launch_tile(const SmallParams& p, bool ta, bool tb, cudaStream_t s) {
  const dim3 grid((p.n + TN - 1) / TN, (p.m + TM - 1) / TM);
  if (!ta && !tb) k_sgemm_small<TM, TN, false, false><<<grid, kSmallThreads, 0, s>>>(p);
  else if (!ta && tb) k_sgemm_small<TM, TN, false, true><<<grid, kSmallThreads, 0, s>>>(p);
  else if (ta && !tb) k_sgemm_small<TM, TN, true, false><<<grid, kSmallThreads, 0, s>>>(p);
  else k_sgemm_small<TM, TN, true, true><<<grid, kSmallThreads, 0, s>>>(p);
}

}  // namespace

bool small_fits(int64_t m, int64_t n, int64_t k) {
  // grid.y <= 65535 tiles of >= 32 rows; int indices
  return m <= 32LL * 65535 && n <= INT32_MAX / 2 && k <= INT32_MAX / 2 && m <= INT32_MAX / 2;
}

tm_status launch_small(const GemmArgs& a, cudaStream_t stream) {
  if (!small_fits(a.m, a.n, a.k)) return TM_ERR_INVALID_VALUE;
  SmallParams p{a.A, a.B, a.C, a.lda, a.ldb, a.ldc, static_cast<int>(a.m), static_cast<int>(a.n),
                static_cast<int>(a.k), a.alpha, a.beta};
  // 32 x 32 tiles while they leave SMs idle, else 64 x 64 (4x the FMAs per
  // loaded element; 2x fewer CTAs than SMs at most)
  const int64_t tiles32 = ((a.m + 31) / 32) * ((a.n + 31) / 32);
  if (tiles32 <= 2 * 148) launch_tile<32, 32>(p, a.ta, a.tb, stream);
  else launch_tile<64, 64>(p, a.ta, a.tb, stream);
  return cudaGetLastError() == cudaSuccess ? TM_OK : TM_ERR_CUDA;
}

}  // namespace tmk
