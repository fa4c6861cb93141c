// simt_gemm.cu -- pure-FP32 SIMT sgemm (validation path) and the C = beta*C
// special-case kernel.
//
// C = alpha*A*B + beta*C with FFMA accumulation in fp32.
// The paper's GPU gemm optimisations: two-level tiling (CTA
// tile 128x128, per-thread 8x8 register block -- "register blocking"),
// shared-memory staging with double buffering ("data movement between global,
// shared and register memory", "data prefetching"), coalesced/vectorised
// global accesses, and an explicit full-tile / partial-tile split in the
// loads and in the fused alpha/beta epilogue ("separate partial tiles from
// full tiles").
#include <cuda_runtime.h>

#include <cstdint>

#include "tm_internal.h"

namespace tmk {

namespace {

constexpr int SBM = 128, SBN = 128, SBK = 8, STHREADS = 256;

struct SimtParams {
  int64_t m, n, k;
  float alpha, beta;
  const float* __restrict__ A;
  int64_t lda;
  const float* __restrict__ B;
  int64_t ldb;
  float* __restrict__ C;
  int64_t ldc;
  int64_t tiles_n;
  bool vec_c;  // C 16-B aligned and ldc % 4 == 0
};

template <bool VEC>
__device__ __forceinline__ void load_a(const SimtParams& p, int64_t row, int64_t kq, float (&v)[4]) {
  // 4 consecutive k of one row of A
  if (VEC && row < p.m && kq + 3 < p.k) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p.A + row * p.lda + kq));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (row < p.m && kq + i < p.k) ? __ldg(p.A + row * p.lda + kq + i) : 0.0f;
  }
}

template <bool VEC>
__device__ __forceinline__ void load_b(const SimtParams& p, int64_t krow, int64_t col, float (&v)[4]) {
  // 4 consecutive columns of one row of B
  if (VEC && krow < p.k && col + 3 < p.n) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p.B + krow * p.ldb + col));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (krow < p.k && col + i < p.n) ? __ldg(p.B + krow * p.ldb + col + i) : 0.0f;
  }
}

template <bool VEC>
__global__ void __launch_bounds__(STHREADS, 2) k_sgemm_simt(SimtParams p) {
  __shared__ __align__(16) float As[2][SBK][SBM + 4];  // k-major copy of the A tile
  __shared__ __align__(16) float Bs[2][SBK][SBN];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t bm = blockIdx.x / p.tiles_n, bn = blockIdx.x % p.tiles_n;
  const int64_t row0 = bm * SBM, col0 = bn * SBN;

  const int a_r = tid >> 1, a_k = (tid & 1) * 4;   // A: 128 rows x 8 k
  const int b_k = tid >> 5, b_c = (tid & 31) * 4;  // B: 8 k x 128 cols

  float ar[4], br[4];
  const int64_t nk = (p.k + SBK - 1) / SBK;

  load_a<VEC>(p, row0 + a_r, a_k, ar);
  load_b<VEC>(p, b_k, col0 + b_c, br);
#pragma unroll
  for (int i = 0; i < 4; ++i) As[0][a_k + i][a_r] = ar[i];
  *reinterpret_cast<float4*>(&Bs[0][b_k][b_c]) = make_float4(br[0], br[1], br[2], br[3]);
  __syncthreads();

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

  for (int64_t kb = 0; kb < nk; ++kb) {
    const int cur = static_cast<int>(kb & 1);
    const bool more = kb + 1 < nk;
    if (more) {  // prefetch the next K-block into registers while computing this one
      const int64_t k0 = (kb + 1) * SBK;
      load_a<VEC>(p, row0 + a_r, k0 + a_k, ar);
      load_b<VEC>(p, k0 + b_k, col0 + b_c, br);
    }
#pragma unroll
    for (int kk = 0; kk < SBK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][kk][64 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) {
#pragma unroll
      for (int i = 0; i < 4; ++i) As[cur ^ 1][a_k + i][a_r] = ar[i];
      *reinterpret_cast<float4*>(&Bs[cur ^ 1][b_k][b_c]) = make_float4(br[0], br[1], br[2], br[3]);
      __syncthreads();
    }
  }

  // ---------------------------------------------------------------- epilogue
  const bool full_tile = (row0 + SBM <= p.m) && (col0 + SBN <= p.n);
  const float alpha = p.alpha, beta = p.beta;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = row0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t c = col0 + h * 64 + tx * 4;
      float* cp = p.C + r * p.ldc + c;
      if (full_tile && p.vec_c) {  // full tile: unpredicated 16-byte accesses
        float4 o;
        if (beta == 0.0f) {
          o = make_float4(alpha * acc[i][4 * h + 0], alpha * acc[i][4 * h + 1], alpha * acc[i][4 * h + 2],
                          alpha * acc[i][4 * h + 3]);
        } else {
          const float4 c0 = *reinterpret_cast<const float4*>(cp);
          o = make_float4(fmaf(alpha, acc[i][4 * h + 0], beta * c0.x), fmaf(alpha, acc[i][4 * h + 1], beta * c0.y),
                          fmaf(alpha, acc[i][4 * h + 2], beta * c0.z), fmaf(alpha, acc[i][4 * h + 3], beta * c0.w));
        }
        *reinterpret_cast<float4*>(cp) = o;
      } else if (r < p.m) {  // partial tile (or unaligned C): predicated scalar accesses
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (c + j < p.n) {
            const float v = acc[i][4 * h + j];
            cp[j] = (beta == 0.0f) ? alpha * v : fmaf(alpha, v, beta * cp[j]);
          }
        }
      }
    }
  }
}

// C = beta*C (alpha == 0 or k == 0); beta == 0 writes zeros without reading C.
__global__ void k_scale_c(int64_t m, int64_t n, float beta, float* __restrict__ C, int64_t ldc) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx / n, j = idx - i * n;
    float* cp = C + i * ldc + j;
    *cp = (beta == 0.0f) ? 0.0f : beta * *cp;
  }
}

}  // namespace

tm_status launch_simt(const GemmArgs& a, cudaStream_t stream) {
  SimtParams p;
  p.m = a.m; p.n = a.n; p.k = a.k;
  p.alpha = a.alpha; p.beta = a.beta;
  p.A = a.A; p.lda = a.lda; p.B = a.B; p.ldb = a.ldb; p.C = a.C; p.ldc = a.ldc;
  p.tiles_n = (a.n + SBN - 1) / SBN;
  const int64_t tiles = ((a.m + SBM - 1) / SBM) * p.tiles_n;
  if (tiles > INT32_MAX) return TM_ERR_INVALID_VALUE;
  p.vec_c = (reinterpret_cast<uintptr_t>(a.C) % 16 == 0) && (a.ldc % 4 == 0);
  const bool vec = (reinterpret_cast<uintptr_t>(a.A) % 16 == 0) && (reinterpret_cast<uintptr_t>(a.B) % 16 == 0) &&
                   (a.lda % 4 == 0) && (a.ldb % 4 == 0);
  if (vec)
    k_sgemm_simt<true><<<static_cast<unsigned>(tiles), STHREADS, 0, stream>>>(p);
  else
    k_sgemm_simt<false><<<static_cast<unsigned>(tiles), STHREADS, 0, stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? TM_OK : TM_ERR_CUDA;
}

tm_status launch_scale(int64_t m, int64_t n, float beta, float* C, int64_t ldc, cudaStream_t stream) {
  const int64_t total = m * n;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_scale_c<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(m, n, beta, C, ldc);
  return cudaGetLastError() == cudaSuccess ? TM_OK : TM_ERR_CUDA;
}

}  // namespace tmk
