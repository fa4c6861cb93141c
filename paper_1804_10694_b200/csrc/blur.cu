// blur.cu -- the paper's Blur (Fig. 3), the workload of its
// distributed example (Fig. 5 Code 3):
//
//   bx(i,j,c) = (in(i,j,c) + in(i,j+1,c) + in(i,j+2,c)) / 3
//   by(i,j,c) = (bx(i,j,c) + bx(i+1,j,c) + bx(i+2,j,c)) / 3
//   0 <= i < N-2, 0 <= j < M-2, 0 <= c < 3.
//
// Layout: row i of the image is 3M contiguous floats, in(i,j,c) at
// in[i*ldi + 3j + c] (channels interleaved, the paper's lin(i,j,c) whose border
// rows are "M*2*3 contiguous data elements").  On a row flattened
// to q = 3j + c the horizontal stage is a 1-D stencil with taps {q, q+3, q+6},
// so channels need no special handling: output element q of row i is
//   by[i][q] = (bx[i][q] + bx[i+1][q] + bx[i+2][q]) / 3,
//   bx[i][q] = (in[i][q] + in[i][q+3] + in[i][q+6]) / 3,   0 <= q < 3(M-2).
//
// HBM-bound (no data reuse beyond the stencil; 24 bytes of HBM traffic per
// output element).  A warp computes 8 output rows x 120 consecutive q: lane l
// loads the float4 at q = 120 w + 4 l of each of the 10 input rows it needs
// (one coalesced 512-B access per row, 8 floats of halo for the 30 output
// lanes), all ten loads issued before any arithmetic (5 KB in flight per warp),
// and takes the six taps it needs beyond its own four from lanes l+1, l+2 with
// shuffles, so each input byte crosses the LSU once per warp.  bx is computed
// once per input row and kept for three output rows in registers (the paper's
// compute_at of bx inside by, without the redundant
// recomputation of overlapped tiling).  The four warps of a CTA take
// vertically adjacent 8-row bands of the same columns, so the two rows a band
// shares with the next one are L1 hits; CTAs are ordered columns-fastest, so
// the CTAs resident at any time read one compact band of the image (DRAM page
// locality: with tall per-warp strips walking down independently, the
// concurrently open rows scatter over the whole image and the same kernel ran
// at 0.6 of the copy rate).
//
// Arithmetic in fp32 with explicit __fadd_rn/__fmul_rn (never contracted to
// FMA, so every element gets the same bits whatever strip or launch computes
// it); "/ 3" is a multiply by fl(1/3) (|by - R|
// <= ~8u * D, D the mean |in| over the nine taps).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "tm_internal.h"

namespace tmk {
namespace {

constexpr int kBlurWarps = 4;   // warps per CTA, stacked along the rows
constexpr int kBlurThreads = 32 * kBlurWarps;
constexpr int kBlurQ = 120;     // output q per warp (30 lanes x 4)
constexpr int kBlurRows = 8;    // output rows per warp
constexpr float kThird = 1.0f / 3.0f;

// Four floats of one row at q0 (zero beyond the row's Qin = 3M floats).
// VIN == 4: rows 16-B aligned, whole float4s inside the row load as one.
template <int VIN>
__device__ __forceinline__ float4 load_row(const float* __restrict__ p, int64_t q0, int64_t Qin) {
  if (VIN == 4 && q0 + 3 < Qin) return __ldg(reinterpret_cast<const float4*>(p + q0));
  float4 v;
  v.x = q0 < Qin ? __ldg(p + q0) : 0.0f;
  v.y = q0 + 1 < Qin ? __ldg(p + q0 + 1) : 0.0f;
  v.z = q0 + 2 < Qin ? __ldg(p + q0 + 2) : 0.0f;
  v.w = q0 + 3 < Qin ? __ldg(p + q0 + 3) : 0.0f;
  return v;
}

// Four outputs at q0 of one row (the row's last group may be partial).
// Streaming stores: the output is never re-read, keep L2 for the input.
template <int VOUT>
__device__ __forceinline__ void store_out(float* __restrict__ p, int64_t q0, int64_t Q, const float (&o)[4]) {
  if (q0 + 3 < Q) {
    if constexpr (VOUT == 4) {
      __stcs(reinterpret_cast<float4*>(p + q0), make_float4(o[0], o[1], o[2], o[3]));
    } else if constexpr (VOUT == 2) {
      __stcs(reinterpret_cast<float2*>(p + q0), make_float2(o[0], o[1]));
      __stcs(reinterpret_cast<float2*>(p + q0 + 2), make_float2(o[2], o[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) __stcs(p + q0 + e, o[e]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (q0 + e < Q) __stcs(p + q0 + e, o[e]);
  }
}

// grid: x = ceil(Q / 120) CTAs along q, y = ceil(nrows / 32) bands of rows.
// Output rows [i0, i0 + nrows) of `out` (pitch ldo) from input rows
// [i0, i0 + nrows + 2) of `in` (pitch ldi); Q = 3(M-2), Qin = 3M.
template <int VIN, int VOUT>
__global__ void __launch_bounds__(kBlurThreads, 8) k_blur(int64_t i0, int64_t nrows, int64_t Q,
                                                          const float* __restrict__ in, int64_t ldi,
                                                          float* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t r0 = (static_cast<int64_t>(blockIdx.y) * kBlurWarps + (threadIdx.x >> 5)) * kBlurRows;
  if (r0 >= nrows) return;  // warp-uniform
  const int nr = nrows - r0 < kBlurRows ? static_cast<int>(nrows - r0) : kBlurRows;
  const int64_t q0 = static_cast<int64_t>(blockIdx.x) * kBlurQ + 4 * lane;
  const int64_t Qin = Q + 6;
  const float* src = in + (i0 + r0) * ldi;
  float* dst = out + (i0 + r0) * ldo;

  float4 v[kBlurRows + 2];
#pragma unroll
  for (int u = 0; u < kBlurRows + 2; ++u)
    v[u] = u < nr + 2 ? load_row<VIN>(src + u * ldi, q0, Qin) : make_float4(0.f, 0.f, 0.f, 0.f);
  float b0[4], b1[4];  // bx of input rows t-2, t-1
#pragma unroll
  for (int t = 0; t < kBlurRows + 2; ++t) {
    if (t >= nr + 2) break;  // warp-uniform
    float w[10];
    w[0] = v[t].x; w[1] = v[t].y; w[2] = v[t].z; w[3] = v[t].w;
    w[4] = __shfl_down_sync(0xffffffffu, v[t].x, 1);
    w[5] = __shfl_down_sync(0xffffffffu, v[t].y, 1);
    w[6] = __shfl_down_sync(0xffffffffu, v[t].z, 1);
    w[7] = __shfl_down_sync(0xffffffffu, v[t].w, 1);
    w[8] = __shfl_down_sync(0xffffffffu, v[t].x, 2);
    w[9] = __shfl_down_sync(0xffffffffu, v[t].y, 2);
    float bn[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) bn[e] = __fmul_rn(__fadd_rn(__fadd_rn(w[e], w[e + 3]), w[e + 6]), kThird);
    if (t >= 2) {
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] = __fmul_rn(__fadd_rn(__fadd_rn(b0[e], b1[e]), bn[e]), kThird);
      if (lane < kBlurQ / 4) store_out<VOUT>(dst + (t - 2) * ldo, q0, Q, o);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      b0[e] = t >= 1 ? b1[e] : bn[e];
      b1[e] = bn[e];
    }
  }
}

template <int VIN, int VOUT>
tm_status launch(int64_t i0, int64_t nrows, int64_t Q, const float* in, int64_t ldi, float* out, int64_t ldo,
                 dim3 grid, cudaStream_t stream) {
  k_blur<VIN, VOUT><<<grid, kBlurThreads, 0, stream>>>(i0, nrows, Q, in, ldi, out, ldo);
  return cudaGetLastError() == cudaSuccess ? TM_OK : TM_ERR_CUDA;
}

}  // namespace

tm_status launch_blur(int64_t i0, int64_t i1, int64_t M, const float* in, int64_t ldi, float* out, int64_t ldo,
                      int num_sms, cudaStream_t stream) {
  const int64_t nrows = i1 - i0;
  const int64_t Q = 3 * (M - 2);
  if (nrows <= 0 || Q <= 0) return TM_OK;
  const int64_t gx = (Q + kBlurQ - 1) / kBlurQ;
  (void)num_sms;
  if (gx > 0x7fffffff) return TM_ERR_INVALID_VALUE;
  // grid.y is limited to 65535 bands of 32 rows: taller images take several launches
  constexpr int64_t kMaxRows = 65535LL * kBlurRows * kBlurWarps;
  if (nrows > kMaxRows) {
    for (int64_t r = 0; r < nrows; r += kMaxRows) {
      tm_status st = launch_blur(i0 + r, i0 + std::min(nrows, r + kMaxRows), M, in, ldi, out, ldo, num_sms, stream);
      if (st != TM_OK) return st;
    }
    return TM_OK;
  }
  const int64_t gy = (nrows + kBlurRows * kBlurWarps - 1) / (kBlurRows * kBlurWarps);
  const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
  auto al = [](const void* p, unsigned a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; };
  const bool vin = al(in, 16) && ldi % 4 == 0;
  const int vout = (al(out, 16) && ldo % 4 == 0) ? 4 : (al(out, 8) && ldo % 2 == 0) ? 2 : 1;
  if (vin) {
    if (vout == 4) return launch<4, 4>(i0, nrows, Q, in, ldi, out, ldo, grid, stream);
    if (vout == 2) return launch<4, 2>(i0, nrows, Q, in, ldi, out, ldo, grid, stream);
    return launch<4, 1>(i0, nrows, Q, in, ldi, out, ldo, grid, stream);
  }
  if (vout == 4) return launch<1, 4>(i0, nrows, Q, in, ldi, out, ldo, grid, stream);
  if (vout == 2) return launch<1, 2>(i0, nrows, Q, in, ldi, out, ldo, grid, stream);
  return launch<1, 1>(i0, nrows, Q, in, ldi, out, ldo, grid, stream);
}

}  // namespace tmk

namespace {
bool blur_args_ok(int64_t N, int64_t M, const float* in, int64_t ldi, const float* out, int64_t ldo) {
  if (N < 3 || M < 3 || !in || !out || ldi < 3 * M || ldo < 3 * (M - 2)) return false;
  const uintptr_t i0 = reinterpret_cast<uintptr_t>(in), o0 = reinterpret_cast<uintptr_t>(out);
  const uintptr_t ibytes = static_cast<uintptr_t>(((N - 1) * ldi + 3 * M) * 4);
  const uintptr_t obytes = static_cast<uintptr_t>(((N - 3) * ldo + 3 * (M - 2)) * 4);
  return !(i0 < o0 + obytes && o0 < i0 + ibytes);
}
}  // namespace

extern "C" tm_status tm_blur(int64_t N, int64_t M, const float* in, int64_t ldi, float* out, int64_t ldo,
                             void* stream) {
  if (!blur_args_ok(N, M, in, ldi, out, ldo)) return TM_ERR_INVALID_VALUE;
  int sms = 0;
  tm_status st = tmk::device_sms(&sms);
  if (st != TM_OK) return st;
  return tmk::launch_blur(0, N - 2, M, in, ldi, out, ldo, sms, static_cast<cudaStream_t>(stream));
}
