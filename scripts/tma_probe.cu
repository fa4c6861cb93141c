// TMA load-rate probe (not part of the product): one CTA per SM, one thread
// issuing TMA loads into a ring, one warp releasing stages without compute.
// Measures how fast a single SM's TMA unit lands boxes of different shapes,
// from DRAM (large source) and from L2 (small, re-read source).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I paper_1804_10694_b200/csrc scripts/tma_probe.cu -o scripts/libtmaprobe.so -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "ptx.cuh"

using namespace tmk;

// wait variants: 0 try_wait (default suspend), 1 test_wait spin, 2 try_wait with a 20 ns suspend hint
__device__ __forceinline__ void wait_v(uint64_t* bar, uint32_t parity, int v) {
  const uint32_t a = ptx::smem_u32(bar);
  uint32_t ok = 0;
  if (v == 1) {
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    } while (!ok);
  } else if (v == 2) {
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 20;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    } while (!ok);
  } else {
    ptx::mbar_wait(bar, parity);
  }
}

struct ProbeP {
  int mode;      // 0: 2D box; 1: 1D bulk copy
  int stages;    // ring depth
  int box_bytes; // bytes per load
  int loads;     // loads per CTA
  int rows_per_load, row_tiles;  // 2D: row coordinate advance per load, tiles along rows
  long long bulk_span;           // 1D: bytes of source
  const char* src;
  int wait_variant;
  int pairs;     // independent producer/consumer warp pairs, each with stages/pairs ring slots
};

__global__ void __launch_bounds__(256) k_probe(const __grid_constant__ CUtensorMap tm, ProbeP p) {
  extern __shared__ uint8_t smem_raw_[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * p.box_bytes);
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.stages; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::fence_mbarrier_init();
  }
  __syncthreads();
  const int pair = warp >> 1, ns = p.stages / p.pairs, s0 = pair * ns, nl = p.loads / p.pairs;
  if ((warp & 1) == 0 && ptx::elect_one()) {  // elect: no per-load R2UR waterfall
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < nl; ++i) {
      wait_v(&empty[s0 + s], ph ^ 1, p.wait_variant);
      ptx::mbar_arrive_expect_tx(&full[s0 + s], p.box_bytes);
      const long long li = static_cast<long long>(blockIdx.x) * p.loads + pair * nl + i;
      uint8_t* dst = smem + (s0 + s) * p.box_bytes;
      if (p.mode == 0) {
        const int rt = static_cast<int>((li * 7919) % p.row_tiles);
        ptx::tma_load_2d(dst, &tm, &full[s0 + s], 0, rt * p.rows_per_load);
      } else {
        const long long off = (li * p.box_bytes) % p.bulk_span;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         ptx::smem_u32(dst)),
                     "l"(p.src + off), "r"(p.box_bytes), "r"(ptx::smem_u32(&full[s0 + s]))
                     : "memory");
      }
      if (++s == ns) { s = 0; ph ^= 1; }
    }
  } else if ((warp & 1) == 1 && ptx::elect_one()) {
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < nl; ++i) {
      wait_v(&full[s0 + s], ph, p.wait_variant);
      ptx::mbar_arrive(&empty[s0 + s]);
      if (++s == ns) { s = 0; ph ^= 1; }
    }
  }
  __syncthreads();
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// swz: 0 none, 1 64B, 2 128B.  box = box_cols floats x box_rows rows of a rows x cols fp32 matrix (ld = cols).
extern "C" int run_tma_probe(const void* src, long long rows, long long cols, int mode, int box_cols, int box_rows,
                             int swz, int stages, int loads, int pairs, int ctas_per_sm, int wait_variant, float* ms) {
  static EncodeTiled enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q) !=
        cudaSuccess)
      return 1;
  }
  CUtensorMap tm{};
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 4)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUtensorMapSwizzle sw = swz == 2 ? CU_TENSOR_MAP_SWIZZLE_128B : swz == 1 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  if (mode == 0 && enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(src), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 2;
  ProbeP p{};
  p.mode = mode;
  p.stages = stages;
  p.box_bytes = box_cols * box_rows * 4;
  p.loads = loads;
  p.rows_per_load = box_rows;
  p.row_tiles = static_cast<int>(rows / box_rows);
  p.bulk_span = rows * cols * 4;
  p.src = static_cast<const char*>(src);
  p.pairs = pairs;
  p.wait_variant = wait_variant;
  const int smem = 1024 + stages * p.box_bytes + stages * 16;
  if (cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 3;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * ctas_per_sm;
  k_probe<<<grid, 64 * pairs, smem>>>(tm, p);  // warm
  cudaEventRecord(e0);
  k_probe<<<grid, 64 * pairs, smem>>>(tm, p);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) return 4;
  cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
