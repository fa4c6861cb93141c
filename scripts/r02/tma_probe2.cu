// TMA streaming probe for the C4 access pattern (not part of the product):
// A = m x k fp32 row-major (k = 576: rows 2304 B apart), every CTA streams
// whole 128-row panels K-block by K-block (32 k = 128 B per row) into a ring of
// 8 x 16 KiB slots, as the GEMM's A producer does.  One load covers KC
// consecutive K-blocks: KC = 1 is the GEMM's 2-D box {32, 128}; KC = 2, 4 use a
// 3-D view {32 (k), m (rows), k/32 (K-block)} with box {32, 128, KC} -- the
// same bytes in the same shared-memory layout (KC consecutive SW128 tiles) in
// one instruction, so the KC x 128 B of each row are requested together.
// `issuers` producer lanes (separate warps) take load groups round-robin; one
// releaser warp frees them in order.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I paper_1804_10694_b200/csrc scripts/r02/tma_probe2.cu -o scripts/r02/libtmaprobe2.so
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

using namespace tmk;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

struct P2 {
  int panels, kblocks, kc, issuers;
  int rows;  // rows per load (3-D box {32, rows, kc}); 128 = the GEMM's A box
};

__global__ void __launch_bounds__(192, 1) k_probe2(const __grid_constant__ CUtensorMap t2, const __grid_constant__ CUtensorMap t3, P2 p) {
  extern __shared__ uint8_t smem_raw_[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_) + 1023) & ~uintptr_t(1023));
  constexpr int kSlots = 8, kSlot = 16384;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSlots * kSlot);
  uint64_t* empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lbytes = p.kc * p.rows * 128, groups = kSlots * kSlot / lbytes;
  if (threadIdx.x == 0) {
    for (int i = 0; i < groups; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::fence_mbarrier_init();
  }
  __syncthreads();
  const int loads_per_panel = (p.kblocks / p.kc) * (128 / p.rows);
  int total = 0;
  for (int pn = blockIdx.x; pn < p.panels; pn += gridDim.x) total += loads_per_panel;
  if (warp < p.issuers && ptx::elect_one()) {  // elect: no per-load R2UR waterfall
    int g = 0, own = 0;
    uint32_t ph = 0;
    int i = 0;
    for (int pn = blockIdx.x; pn < p.panels; pn += gridDim.x)
      for (int l = 0; l < loads_per_panel; ++l, ++i) {
        if (own == warp) {
          ptx::mbar_wait(&empty[g], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full[g], p.kc * p.rows * 128);
          uint8_t* dst = smem + g * lbytes;
          const int per_k = 128 / p.rows;  // row groups per K chunk: rows-major when rows < 128
          const int kq = p.rows < 128 ? l / per_k : l, rg = p.rows < 128 ? l % per_k : 0;
          if (p.kc == 1 && p.rows == 128) ptx::tma_load_2d(dst, &t2, &full[g], l * 32, pn * 128);
          else tma_load_3d(dst, &t3, &full[g], 0, pn * 128 + rg * p.rows, kq * p.kc);
        }
        if (++own == p.issuers) own = 0;
        if (++g == groups) { g = 0; ph ^= 1; }
      }
  } else if (warp == 5 && ptx::elect_one()) {
    int g = 0;
    uint32_t ph = 0;
    for (int i = 0; i < total; ++i) {
      ptx::mbar_wait(&full[g], ph);
      ptx::mbar_arrive(&empty[g]);
      if (++g == groups) { g = 0; ph ^= 1; }
    }
  }
  __syncthreads();
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int run_probe2(const float* A, long long m, long long k, int kc, int rows, int issuers, int grid, float* us) {
  static EncodeTiled enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q) != cudaSuccess)
      return 1;
  }
  CUtensorMap t2{}, t3{};
  cuuint64_t d2[2] = {(cuuint64_t)k, (cuuint64_t)m}, s2[1] = {(cuuint64_t)k * 4};
  cuuint32_t b2[2] = {32, 128}, e2[2] = {1, 1};
  if (enc(&t2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 2;
  cuuint64_t d3[3] = {32, (cuuint64_t)m, (cuuint64_t)(k / 32)}, s3[2] = {(cuuint64_t)k * 4, 128};
  cuuint32_t b3[3] = {32, (cuuint32_t)rows, (cuuint32_t)kc}, e3[3] = {1, 1, 1};
  if (enc(&t3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)A, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 3;
  P2 p{static_cast<int>(m / 128), static_cast<int>(k / 32), kc, issuers, rows};
  const int smem = 1024 + 8 * 16384 + 512;
  if (cudaFuncSetAttribute(k_probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 1; ++r) {
    cudaEventRecord(e0);
    k_probe2<<<grid, 192, smem>>>(t2, t3, p);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) return 5;
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  *us = best * 1e3f;
  return cudaGetLastError() == cudaSuccess ? 0 : 6;
}
