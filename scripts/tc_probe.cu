// tc_probe.cu -- bring-up probes for tcgen05 (not part of the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o libtcprobe.so tc_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_1804_10694_b200/csrc/ptx.cuh"

using namespace tmk;

// 1) TMEM store/load round trip: each thread stores (warp*1000 + lane) into
//    column c of its lane and reads it back.
__global__ void probe_tmem(float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) ptx::tmem_alloc<1>(&slot, 32);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = slot;
  const uint32_t taddr = base + ((warp * 32) << 16);
  uint32_t v = __float_as_uint(float(warp * 1000 + lane));
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr + 3), "r"(v) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr + 3));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[threadIdx.x] = __uint_as_float(r);
  out[128 + threadIdx.x] = __uint_as_float(base);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<1>(base, 32);
}

// 2) One MMA M=128 N=32 K=8 from manually filled smem.
//    variant 0: A K-major, B K-major, SWIZZLE_NONE (core matrices 8 rows x 16 B)
//    variant 1: A K-major SW128 (rows of 128 B = 32 k), B MN-major SW128 (rows of 128 B = 32 n)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

struct ProbeCfg {
  int a_mode, b_mode;            // a: 0 K-major none, 1 K-major SW128; b: 0 K-major none, 1 MN-major SW128, 2 MN-major none
  uint32_t a_lbo, a_sbo, a_layout, b_lbo, b_sbo, b_layout, idesc;
};

__global__ void probe_mma(const float* A, const float* B, float* out, ProbeCfg c) {
  // A: 128 x 8 (row-major, lda 8); B: 8 x 32 (row-major, ldb 32); out: 128 x 32
  extern __shared__ __align__(1024) uint8_t sm_[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_ + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)sm;             // 16 KiB
  float* sB = (float*)(sm + 16384);   // 16 KiB
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 4096; i += blockDim.x) { sA[i] = 0.f; sB[i] = 0.f; }
  __syncthreads();
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    int r = i / 8, k = i % 8, off;
    if (c.a_mode == 0) off = (r / 8) * 256 + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4;
    else off = r * 128 + (((k / 4) ^ (r % 8)) * 16) + (k % 4) * 4;
    sA[off / 4] = A[r * 8 + k];
  }
  for (int i = tid; i < 8 * 32; i += blockDim.x) {
    int p = i / 32, n = i % 32, off;
    if (c.b_mode == 0) off = (n / 8) * 256 + (p / 4) * 128 + (n % 8) * 16 + (p % 4) * 4;
    else if (c.b_mode == 1) off = p * 128 + (((n / 4) ^ (p % 8)) * 16) + (n % 4) * 4;
    else if (c.b_mode == 3) off = p * 128 + (((n / 8) ^ (p % 4)) * 32) + (n % 8) * 4;  // SW128 atom 32B
    else off = (n / 4) * 128 + (p % 8) * 16 + (n % 4) * 4;
    sB[off / 4] = B[p * 32 + n];
  }
  ptx::fence_proxy_async_smem();
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbarrier_init(); }
  if (warp == 0) ptx::tmem_alloc<1>(&slot, 32);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = slot;
  if (warp == 1 && ptx::elect_one()) {
    uint64_t ad = sdesc(ptx::smem_u32(sA), c.a_lbo, c.a_sbo, c.a_layout);
    uint64_t bd = sdesc(ptx::smem_u32(sB), c.b_lbo, c.b_sbo, c.b_layout);
    ptx::mma_tf32<1>(base, ad, bd, c.idesc, 0u);
    ptx::mma_commit<1>(&bar);
  }
  __syncwarp();
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  uint32_t r[16];
  for (int cc = 0; cc < 2; ++cc) {
    ptx::tmem_ld_32x32b_x16(base + ((warp * 32) << 16) + cc * 16, r);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(warp * 32 + lane) * 32 + cc * 16 + j] = __uint_as_float(r[j]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<1>(base, 32);
}

extern "C" int run_probe_tmem(float* out) {
  probe_tmem<<<1, 128>>>(out);
  return (int)cudaDeviceSynchronize();
}

extern "C" int run_probe_mma(const float* A, const float* B, float* out, const ProbeCfg* c) {
  cudaFuncSetAttribute(probe_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  probe_mma<<<1, 128, 40 * 1024>>>(A, B, out, *c);
  return (int)cudaDeviceSynchronize();
}

// bf16 variant: A 128x16, B 16x32 (bf16 given as uint16 bit patterns), kind::f16.
__global__ void probe_mma_bf16(const uint16_t* A, const uint16_t* B, float* out, ProbeCfg c) {
  extern __shared__ __align__(1024) uint8_t sm_[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_ + 1023) & ~(uintptr_t)1023);
  uint16_t* sA = (uint16_t*)sm;
  uint16_t* sB = (uint16_t*)(sm + 16384);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 8192; i += blockDim.x) { sA[i] = 0; sB[i] = 0; }
  __syncthreads();
  for (int i = tid; i < 128 * 16; i += blockDim.x) {
    int r = i / 16, k = i % 16, off;
    off = (r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
    sA[off / 2] = A[r * 16 + k];
  }
  for (int i = tid; i < 16 * 32; i += blockDim.x) {
    int p = i / 32, n = i % 32, off;
    if (c.b_mode == 0) off = (n / 8) * 256 + (p / 8) * 128 + (n % 8) * 16 + (p % 8) * 2;
    else if (c.b_mode == 1) off = (p / 8) * 1024 + (p % 8) * 128 + (((n / 8) ^ (p % 8)) * 16) + (n % 8) * 2;
    else off = (n / 8) * 128 + (p / 8) * 512 + (p % 8) * 16 + (n % 8) * 2;
    sB[off / 2] = B[p * 32 + n];
  }
  ptx::fence_proxy_async_smem();
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbarrier_init(); }
  if (warp == 0) ptx::tmem_alloc<1>(&slot, 32);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = slot;
  if (warp == 1 && ptx::elect_one()) {
    uint64_t ad = sdesc(ptx::smem_u32(sA), c.a_lbo, c.a_sbo, c.a_layout);
    uint64_t bd = sdesc(ptx::smem_u32(sB), c.b_lbo, c.b_sbo, c.b_layout);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(base), "l"(ad), "l"(bd), "r"(c.idesc), "r"(0u) : "memory");
    ptx::mma_commit<1>(&bar);
  }
  __syncwarp();
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  uint32_t r[16];
  for (int cc = 0; cc < 2; ++cc) {
    ptx::tmem_ld_32x32b_x16(base + ((warp * 32) << 16) + cc * 16, r);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(warp * 32 + lane) * 32 + cc * 16 + j] = __uint_as_float(r[j]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<1>(base, 32);
}

extern "C" int run_probe_mma_bf16(const uint16_t* A, const uint16_t* B, float* out, const ProbeCfg* c) {
  cudaFuncSetAttribute(probe_mma_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  probe_mma_bf16<<<1, 128, 40 * 1024>>>(A, B, out, *c);
  return (int)cudaDeviceSynchronize();
}
