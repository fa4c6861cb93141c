// tm_internal.h -- internal interfaces between the C-ABI layer and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/tm.h"

namespace tmk {

// The dynamic-shared-memory opt-in (cudaFuncSetAttribute) is recorded per
// device, so it is set once per (kernel, device): `done` is the caller's
// per-kernel bitmask of devices already opted in (devices >= 64 set it every
// call).  Thread-safe: a race only repeats the idempotent attribute call.
template <class Kernel>
tm_status ensure_smem_optin(std::atomic<unsigned long long>& done, Kernel kern, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TM_ERR_CUDA;
  const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return TM_OK;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return TM_ERR_CUDA;
  done.fetch_or(bit, std::memory_order_release);
  return TM_OK;
}

// The current device's SM count, after checking it is an sm_100 part
// (TM_ERR_UNSUPPORTED_DEVICE otherwise; api.cpp).
tm_status device_sms(int* sms);

// C = alpha * op(A) * op(B) + beta * C, row-major.  ta: op(A) = A^T (A stored
// k x m, lda >= m); tb: op(B) = B^T (B stored n x k, ldb >= k).
struct GemmArgs {
  int64_t m, n, k;
  float alpha, beta;
  const float* A;
  int64_t lda;
  const float* B;
  int64_t ldb;
  float* C;
  int64_t ldc;
  bool ta = false, tb = false;
  // Fused distributed mode (dist.cpp): B arrives in K-chunks of kchunk rows
  // while the GEMM runs; chunk c is present once kflags[c] >= kepoch (written
  // by the transfer stream).  Tensor-core path only (kflags == nullptr: none).
  const unsigned* kflags = nullptr;
  unsigned kepoch = 0;
  int64_t kchunk = 0;
};

// Tensor-core configuration: CTA group (1 or 2), B columns per CTA (32/64/128),
// precision variant (tc_gemm.cuh kPrec*: 0 = 1xTF32, 1 = 3xTF32, 2 = BF16x9).
struct TcChoice {
  int cg;
  int bn_cta;
  int prec;
  bool streamk;  // stream-K decomposition (wave-quantized shapes)
};

template <bool TA, bool TB>
tm_status launch_tc_op(const GemmArgs& a, const TcChoice& c, int num_sms, cudaStream_t stream);
inline tm_status launch_tc(const GemmArgs& a, const TcChoice& c, int num_sms, cudaStream_t stream) {
  if (!a.ta && !a.tb) return launch_tc_op<false, false>(a, c, num_sms, stream);
  if (!a.ta && a.tb) return launch_tc_op<false, true>(a, c, num_sms, stream);
  if (a.ta && !a.tb) return launch_tc_op<true, false>(a, c, num_sms, stream);
  return launch_tc_op<true, true>(a, c, num_sms, stream);
}
tm_status launch_simt(const GemmArgs& a, cudaStream_t stream);
// Latency-bound small problems (small_gemm.cu): FP32 FFMA, one CTA per 32x32
// or 64x64 tile.  small_fits: the index ranges it supports.
bool small_fits(int64_t m, int64_t n, int64_t k);
tm_status launch_small(const GemmArgs& a, cudaStream_t stream);
tm_status launch_scale(int64_t m, int64_t n, float beta, float* C, int64_t ldc, cudaStream_t stream);
// Reads `bytes` (a multiple of 16) of `buf` to evict L2 between timed runs (tune.cpp).
tm_status launch_l2_flush(const float* buf, int64_t bytes, cudaStream_t stream);

// tm_sgemm with `sm_reserve` SMs left free (distributed mode, so the NCCL
// broadcast kernels can run concurrently with the persistent GEMM).  With
// a.kflags set (fused distributed mode) it runs the tensor-core path only.
tm_status sgemm_reserve(const GemmArgs& a, cudaStream_t stream, int sm_reserve);

// Library-owned stream-K workspace for `stream` on the current device: at least
// ws_bytes of fp32 partials and flag_count epoch flags; *epoch is the value this
// launch must write (flags hold earlier epochs, never the new one).  Under CUDA
// graph capture the workspace is allocated inside the graph and *graph_owned is
// set: the caller enqueues cudaFreeAsync(*graph_owned, stream) after its launch.
tm_status streamk_workspace(cudaStream_t stream, size_t ws_bytes, size_t flag_count, float** ws, unsigned** flags,
                            unsigned* epoch, void** graph_owned);

// Implicit-GEMM convolution, NHWC activations, KRSC filters, stride 1:
// Y[b,y,x,f] = alpha * sum X[b, y+ky-pad, x+kx-pad, c] * Wt[f,ky,kx,c] + beta * Y.
struct ConvArgs {
  int64_t nb, h, w, c, f, r, s, pad;
  float alpha, beta;
  const float* X;
  const float* Wt;
  float* Y;
#ifdef __CUDACC__
  __host__ __device__
#endif
  int64_t ho() const { return h + 2 * pad - r + 1; }
#ifdef __CUDACC__
  __host__ __device__
#endif
  int64_t wo() const { return w + 2 * pad - s + 1; }
};
// bk: channels per stage (16 or 32); cg/bn as TcChoice.
tm_status launch_conv_tc(const ConvArgs& a, int cg, int bn, int bk, bool streamk, int num_sms, cudaStream_t stream);
tm_status launch_conv_simt(const ConvArgs& a, cudaStream_t stream);
// Direct (halo-tile) tensor-core convolution for C % 16 == 0, F <= 64 and
// filters that fit in shared memory (tc_conv_direct.cu).
bool conv_direct_fits(const ConvArgs& a);
// Launches the direct kernel takes for this shape: 1, 2 (filter columns split
// over two launches), or 0 (does not fit).
int conv_direct_launches(const ConvArgs& a);
tm_status launch_conv_direct(const ConvArgs& a, int num_sms, cudaStream_t stream);

// Measured-configuration cache (tune.cpp): the tuned choice for this problem
// shape on `sms` SMs, if tm_sgemm_tune (or tm_tune_cache_load) recorded one.
bool tune_lookup(const GemmArgs& a, int sms, TcChoice* out);
// Whether tm_sgemm_op(..., TM_ALGO_TF32X3) would accept these arguments (host-only).
bool tc_plan_ok(const GemmArgs& a);

// Stream memory operations (dist.cpp; driver entry points, no SM): write
// *flag = value after all earlier work of `s`; make `s` wait until
// (int32)(*flag - value) >= 0.  flag may be peer memory (IPC-mapped).
tm_status stream_write_u32(cudaStream_t s, unsigned* flag, unsigned value);
tm_status stream_wait_u32(cudaStream_t s, const unsigned* flag, unsigned value);
// Base and size of the device allocation containing p (cuMemGetAddressRange).
tm_status device_allocation(const void* p, void** base, size_t* bytes);
// SMs the distributed schedules leave to NCCL kernels (TM_DIST_COMM_SMS).
int dist_comm_ctas();

// Blur (blur.cu): output rows [i0, i1) of the two-stage
// 3x3 box blur of an image with N rows of 3M floats (pitch ldi), into out rows
// [i0, i1) (pitch ldo).  The rows needed from `in` are [i0, i1 + 2).
tm_status launch_blur(int64_t i0, int64_t i1, int64_t M, const float* in, int64_t ldi, float* out, int64_t ldo,
                      int num_sms, cudaStream_t stream);

// Picks the tensor-core configuration for a shape (planner, plan.cpp).
TcChoice plan_tc(int64_t m, int64_t n, int64_t k, int num_sms);
// Whether a configuration should run stream-K for this shape.
bool plan_streamk(int64_t m, int64_t n, int64_t k, int cg, int bn_cta, int num_sms);
int64_t streamk_region(int64_t num_tiles, int64_t kblocks, int clusters, int mode, int* clusters_used);

}  // namespace tmk
