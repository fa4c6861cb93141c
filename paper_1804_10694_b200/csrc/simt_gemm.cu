// simt_gemm.cu -- pure-FP32 SIMT sgemm (validation path) and the C = beta*C
// special-case kernel.
//
// C = alpha*op(A)*op(B) + beta*C (op = transposes)
// with FFMA accumulation in fp32.
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

// 4 consecutive elements [inner, inner+4) of row `outer` of a row-major array
// (leading dimension ld), zero outside [0, outer_lim) x [0, inner_lim).
template <bool VEC>
__device__ __forceinline__ void load4(const float* __restrict__ X, int64_t ld, int64_t outer, int64_t outer_lim,
                                      int64_t inner, int64_t inner_lim, float (&v)[4]) {
  if (VEC && outer < outer_lim && inner + 3 < inner_lim) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(X + outer * ld + inner));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (outer < outer_lim && inner + i < inner_lim) ? __ldg(X + outer * ld + inner + i) : 0.0f;
  }
}

// TA: op(A) = A^T (A stored k x m); TB: op(B) = B^T (B stored n x k).
template <bool VEC, bool TA, bool TB>
__global__ void __launch_bounds__(STHREADS, 2) k_sgemm_simt(SimtParams p) {
  __shared__ __align__(16) float As[2][SBK][SBM + 4];  // k-major copy of the A tile
  __shared__ __align__(16) float Bs[2][SBK][SBN];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t bm = blockIdx.x / p.tiles_n, bn = blockIdx.x % p.tiles_n;
  const int64_t row0 = bm * SBM, col0 = bn * SBN;

  // Global -> register mapping (each thread loads 4 contiguous elements):
  //   A  (m x k, K contiguous):  row tid/2,        k (tid%2)*4..+3   -> transposed smem stores
  //   A^T(k x m, M contiguous):  k tid/32,         rows (tid%32)*4   -> one 16-B smem store
  //   B  (k x n, N contiguous):  k tid/32,         cols (tid%32)*4   -> one 16-B smem store
  //   B^T(n x k, K contiguous):  col tid/2,        k (tid%2)*4..+3   -> transposed smem stores
  const int a_o = TA ? (tid >> 5) : (tid >> 1), a_i = TA ? (tid & 31) * 4 : (tid & 1) * 4;
  const int b_o = TB ? (tid >> 1) : (tid >> 5), b_i = TB ? (tid & 1) * 4 : (tid & 31) * 4;

  float ar[4], br[4];
  const int64_t nk = (p.k + SBK - 1) / SBK;
  auto load_tiles = [&](int64_t k0) {
    if (TA) load4<VEC>(p.A, p.lda, k0 + a_o, p.k, row0 + a_i, p.m, ar);
    else load4<VEC>(p.A, p.lda, row0 + a_o, p.m, k0 + a_i, p.k, ar);
    if (TB) load4<VEC>(p.B, p.ldb, col0 + b_o, p.n, k0 + b_i, p.k, br);
    else load4<VEC>(p.B, p.ldb, k0 + b_o, p.k, col0 + b_i, p.n, br);
  };
  auto store_tiles = [&](int buf) {
    if (TA) {
      *reinterpret_cast<float4*>(&As[buf][a_o][a_i]) = make_float4(ar[0], ar[1], ar[2], ar[3]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) As[buf][a_i + i][a_o] = ar[i];
    }
    if (TB) {
#pragma unroll
      for (int i = 0; i < 4; ++i) Bs[buf][b_i + i][b_o] = br[i];
    } else {
      *reinterpret_cast<float4*>(&Bs[buf][b_o][b_i]) = make_float4(br[0], br[1], br[2], br[3]);
    }
  };

  load_tiles(0);
  store_tiles(0);
  __syncthreads();

  // Accumulators as column pairs for the packed FP32 FMA (fma.rn.f32x2 =
  // FFMA2: two independent round-to-nearest FMAs per instruction, so the
  // results are identical to scalar FFMA with half the issue slots).
  unsigned long long acc2[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;

  for (int64_t kb = 0; kb < nk; ++kb) {
    const int cur = static_cast<int>(kb & 1);
    const bool more = kb + 1 < nk;
    if (more) load_tiles((kb + 1) * SBK);  // prefetch the next K-block into registers while computing this one
#pragma unroll
    for (int kk = 0; kk < SBK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][kk][64 + ty * 4]);
      const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(&Bs[cur][kk][tx * 4]);
      const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(&Bs[cur][kk][64 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const unsigned long long bp[4] = {b0.x, b0.y, b1.x, b1.y};  // column pairs (j, j+1)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        unsigned long long ap;
        asm("mov.b64 %0, {%1, %1};" : "=l"(ap) : "f"(av[i]));
#pragma unroll
        for (int j = 0; j < 4; ++j) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[i][j]) : "l"(ap), "l"(bp[j]));
      }
    }
    if (more) {
      store_tiles(cur ^ 1);
      __syncthreads();
    }
  }

  // ---------------------------------------------------------------- epilogue
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i][2 * j]), "=f"(acc[i][2 * j + 1]) : "l"(acc2[i][j]));
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

// L2 eviction for the tuner's timings: reads `n` float4 (no dirty lines left
// behind, unlike a write-flush); the sum is stored only if it is NaN-like,
// which never happens for the zero-filled buffer but keeps the loads live.
__global__ void k_l2_flush(const float4* __restrict__ buf, int64_t n, float* sink) {
  float acc = 0.0f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = __ldcs(buf + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc != acc) *sink = acc;
}

// Direct NHWC / KRSC convolution, FP32 FFMA (validation path for the
// implicit-GEMM tensor-core kernel and fallback for any shape): one thread per
// output pixel, 16 filters per thread; the group's filter taps are staged in
// shared memory per (ky, kx) in chunks of kConvCc channels (any C fits), and
// filter groups stride over gridDim.y (any F fits).  Summation order per output:
// ky, kx, c ascending (chunking does not reorder it).
constexpr int kConvF = 16;
constexpr int kConvCc = 512;
__global__ void __launch_bounds__(128) k_conv_simt(ConvArgs a) {
  __shared__ float wsh[kConvF * kConvCc];  // [kConvF][cc] filters of one tap, one channel chunk
  const int64_t ho = a.ho(), wo = a.wo();
  const int64_t P = a.nb * ho * wo;
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t fgroups = (a.f + kConvF - 1) / kConvF;
  int64_t b = 0, y = 0, x = 0;
  if (q < P) {
    b = q / (ho * wo);
    y = (q / wo) % ho;
    x = q % wo;
  }
  for (int64_t fg = blockIdx.y; fg < fgroups; fg += gridDim.y) {
    const int64_t f0 = fg * kConvF;
    const int nf = static_cast<int>(a.f - f0 < kConvF ? a.f - f0 : kConvF);
    float acc[kConvF];
#pragma unroll
    for (int j = 0; j < kConvF; ++j) acc[j] = 0.0f;
    for (int64_t ky = 0; ky < a.r; ++ky) {
      for (int64_t kx = 0; kx < a.s; ++kx) {
        for (int64_t c0 = 0; c0 < a.c; c0 += kConvCc) {
          const int64_t cc = a.c - c0 < kConvCc ? a.c - c0 : kConvCc;
          __syncthreads();
          for (int64_t i = threadIdx.x; i < static_cast<int64_t>(nf) * cc; i += blockDim.x) {
            const int64_t fj = i / cc, c = i - fj * cc;
            wsh[fj * cc + c] = a.Wt[(((f0 + fj) * a.r + ky) * a.s + kx) * a.c + c0 + c];
          }
          __syncthreads();
          const int64_t iy = y + ky - a.pad, ix = x + kx - a.pad;
          if (q < P && iy >= 0 && iy < a.h && ix >= 0 && ix < a.w) {
            const float* xp = a.X + ((b * a.h + iy) * a.w + ix) * a.c + c0;
            for (int64_t c = 0; c < cc; ++c) {
              const float xv = __ldg(xp + c);
#pragma unroll
              for (int j = 0; j < kConvF; ++j)
                if (j < nf) acc[j] = fmaf(xv, wsh[j * cc + c], acc[j]);
            }
          }
        }
      }
    }
    if (q < P) {
      float* yp = a.Y + q * a.f + f0;
#pragma unroll
      for (int j = 0; j < kConvF; ++j)
        if (j < nf) yp[j] = (a.beta == 0.0f) ? a.alpha * acc[j] : fmaf(a.alpha, acc[j], a.beta * yp[j]);
    }
  }
}

}  // namespace

tm_status launch_conv_simt(const ConvArgs& a, cudaStream_t stream) {
  const int64_t P = a.nb * a.ho() * a.wo();
  const int64_t blocks = (P + 127) / 128;
  const int64_t fgroups = (a.f + kConvF - 1) / kConvF;
  if (blocks > INT32_MAX) return TM_ERR_INVALID_VALUE;
  const unsigned gy = static_cast<unsigned>(fgroups < 65535 ? fgroups : 65535);
  k_conv_simt<<<dim3(static_cast<unsigned>(blocks), gy), 128, 0, stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? TM_OK : TM_ERR_CUDA;
}

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
  const unsigned g = static_cast<unsigned>(tiles);
  const int v = (vec ? 4 : 0) | (a.ta ? 2 : 0) | (a.tb ? 1 : 0);
  switch (v) {
    case 0: k_sgemm_simt<false, false, false><<<g, STHREADS, 0, stream>>>(p); break;
    case 1: k_sgemm_simt<false, false, true><<<g, STHREADS, 0, stream>>>(p); break;
    case 2: k_sgemm_simt<false, true, false><<<g, STHREADS, 0, stream>>>(p); break;
    case 3: k_sgemm_simt<false, true, true><<<g, STHREADS, 0, stream>>>(p); break;
    case 4: k_sgemm_simt<true, false, false><<<g, STHREADS, 0, stream>>>(p); break;
    case 5: k_sgemm_simt<true, false, true><<<g, STHREADS, 0, stream>>>(p); break;
    case 6: k_sgemm_simt<true, true, false><<<g, STHREADS, 0, stream>>>(p); break;
    default: k_sgemm_simt<true, true, true><<<g, STHREADS, 0, stream>>>(p); break;
  }
  return cudaGetLastError() == cudaSuccess ? TM_OK : TM_ERR_CUDA;
}

tm_status launch_l2_flush(const float* buf, int64_t bytes, cudaStream_t stream) {
  k_l2_flush<<<148 * 8, 256, 0, stream>>>(reinterpret_cast<const float4*>(buf), bytes / 16,
                                          const_cast<float*>(buf));
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
