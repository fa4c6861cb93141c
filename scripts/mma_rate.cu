// tcgen05 kind::tf32 issue/throughput probe (not part of the product): one CTA
// per SM, one thread issues `reps` MMAs (M = 128, cta_group::1, N given, K = 8)
// accumulating into one TMEM tile, then commits and waits.  A from shared
// memory (K-major SW128 descriptor) or from TMEM; operand values are zero (the
// rate does not depend on them).  Reports cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I paper_1804_10694_b200/csrc scripts/mma_rate.cu -o scripts/libmmarate.so
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

using namespace tmk;
__device__ __forceinline__ bool lane_is0() { return (threadIdx.x & 31) == 0; }

__global__ void __launch_bounds__(128, 1) k_rate(int n, int a_tmem, int reps, int n_acc, int m, int bsw, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw_[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 96 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) ptx::sts128(ptx::smem_u32(smem) + i * 16, make_uint4(0, 0, 0, 0));
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbarrier_init();
  }
  ptx::fence_proxy_async_smem();
  if (warp == 0) ptx::tmem_alloc<1>(slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 1 && n_acc < 0) {
    // whole warp runs the issue loop (operands stay warp-uniform: uniform
    // registers, no R2UR); one elected lane issues each MMA
    const uint32_t idesc = ptx::idesc_tf32(m, n, 0, 0);
    const uint64_t ad = ptx::sdesc(ptx::smem_u32(smem), 16, 1024, ptx::kLayoutSW128);
    const uint64_t bd = ptx::sdesc(ptx::smem_u32(smem + 32 * 1024), 16, 1024, ptx::kLayoutSW128);
    const uint32_t a_t = tmem + 256 + 128;
    const int na = -n_acc;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = tmem + static_cast<uint32_t>((r % na) * n);
      if (ptx::elect_one()) {
        if (a_tmem) ptx::mma_tf32_tmem_a<1>(d, a_t + (r & 3) * 8, bd + 2 * (r & 3), idesc, 1u);
        else ptx::mma_tf32<1>(d, ad + 2 * (r & 3), bd + 2 * (r & 3), idesc, 1u);
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (ptx::elect_one()) ptx::mma_commit<1>(bar);
    __syncwarp();
    ptx::mbar_wait(bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0 && lane_is0()) {
      out[0] = static_cast<unsigned long long>(t1 - t0);
      out[1] = static_cast<unsigned long long>(t2 - t0);
    }
  } else if (warp == 1 && n_acc >= 0 && ptx::elect_one()) {  // elect: the compiler then knows one lane issues (no per-MMA R2UR waterfall)
    const uint32_t idesc = ptx::idesc_tf32(m, n, 0, 0);
    const uint64_t ad = ptx::sdesc(ptx::smem_u32(smem), 16, 1024, ptx::kLayoutSW128);
    const uint64_t bd = bsw == 64 ? ptx::sdesc(ptx::smem_u32(smem + 32 * 1024), 16, 512, ptx::kLayoutSW64)
                                  : ptx::sdesc(ptx::smem_u32(smem + 32 * 1024), 16, 1024, ptx::kLayoutSW128);
    const uint32_t a_t = tmem + 256 + 128;  // A in TMEM columns 384.. (8 per K step)
    long long t0 = clock64();
    if (n_acc == 0) {
      // lean issue: everything loop-invariant, 8 MMAs per iteration
      const uint64_t b0 = bd, b1 = bd + 2, b2 = bd + 4, b3 = bd + 6;
      if (a_tmem) {
        for (int r = 0; r < reps; r += 8) {
          ptx::mma_tf32_tmem_a<1>(tmem, a_t, b0, idesc, 1u);
          ptx::mma_tf32_tmem_a<1>(tmem, a_t + 8, b1, idesc, 1u);
          ptx::mma_tf32_tmem_a<1>(tmem, a_t + 16, b2, idesc, 1u);
          ptx::mma_tf32_tmem_a<1>(tmem, a_t + 24, b3, idesc, 1u);
          ptx::mma_tf32_tmem_a<1>(tmem, a_t, b0, idesc, 1u);
          ptx::mma_tf32_tmem_a<1>(tmem, a_t + 8, b1, idesc, 1u);
          ptx::mma_tf32_tmem_a<1>(tmem, a_t + 16, b2, idesc, 1u);
          ptx::mma_tf32_tmem_a<1>(tmem, a_t + 24, b3, idesc, 1u);
        }
      } else {
        const uint64_t a0 = ad, a1 = ad + 2, a2 = ad + 4, a3 = ad + 6;
        for (int r = 0; r < reps; r += 8) {
          ptx::mma_tf32<1>(tmem, a0, b0, idesc, 1u);
          ptx::mma_tf32<1>(tmem, a1, b1, idesc, 1u);
          ptx::mma_tf32<1>(tmem, a2, b2, idesc, 1u);
          ptx::mma_tf32<1>(tmem, a3, b3, idesc, 1u);
          ptx::mma_tf32<1>(tmem, a0, b0, idesc, 1u);
          ptx::mma_tf32<1>(tmem, a1, b1, idesc, 1u);
          ptx::mma_tf32<1>(tmem, a2, b2, idesc, 1u);
          ptx::mma_tf32<1>(tmem, a3, b3, idesc, 1u);
        }
      }
    } else {
      for (int r = 0; r < reps; ++r) {
        const uint32_t d = tmem + static_cast<uint32_t>((r % n_acc) * n);
        if (a_tmem) ptx::mma_tf32_tmem_a<1>(d, a_t + (r & 3) * 8, bd + 2 * (r & 3), idesc, 1u);
        else ptx::mma_tf32<1>(d, ad + 2 * (r & 3), bd + 2 * (r & 3), idesc, 1u);
      }
    }
    long long t1 = clock64();
    ptx::mma_commit<1>(bar);
    ptx::mbar_wait(bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = static_cast<unsigned long long>(t1 - t0);
      out[1] = static_cast<unsigned long long>(t2 - t0);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem, 512);
  }
}

extern "C" int run_mma_rate(int n, int a_tmem, int reps, int n_acc, int m, int bsw, unsigned long long* issue_cycles,
                            unsigned long long* total_cycles, float* ms) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int smem = 96 * 1024 + 2048;
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_rate<<<148, 128, smem>>>(n, a_tmem, reps, n_acc, m, bsw, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<<<148, 128, smem>>>(n, a_tmem, reps, n_acc, m, bsw, d);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) return 1;
  cudaEventElapsedTime(ms, e0, e1);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  *issue_cycles = h[0];
  *total_cycles = h[1];
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
