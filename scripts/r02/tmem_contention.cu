// Does tcgen05.st / tcgen05.ld traffic from other warps slow tcgen05.mma?  (not
// part of the product; explains the direct convolution's MMA rate)
// One CTA per SM, 256 threads: warp 0 allocates TMEM; one lane of warp 1 issues
// `reps` kind::tf32 MMAs (M = 128, N given, A from TMEM columns 448.., B from
// shared memory SW64, D at column 0); warps 4-7 (one warpgroup, all four TMEM
// lane quarters) meanwhile loop tcgen05.st.32x32b.x32 (mode 1) or
// tcgen05.ld.32x32b.x16 (mode 2) on columns 256..383, or shared-memory
// 16-B loads (mode 3), or tcgen05.st into the MMAs' own A columns 448..479
// (mode 4, racy values, timing only), until the MMAs finish.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I paper_1804_10694_b200/csrc scripts/r02/tmem_contention.cu -o scripts/r02/libtmemcont.so
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

using namespace tmk;

__global__ void __launch_bounds__(256, 1) k_cont(int n, int reps, int mode, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw_[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 64 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 6);
  volatile int* done = reinterpret_cast<volatile int*>(bar + 7);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) ptx::sts128(ptx::smem_u32(smem) + i * 16, make_uint4(0, 0, 0, 0));
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbarrier_init();
    *done = 0;
  }
  ptx::fence_proxy_async_smem();
  if (warp == 0) ptx::tmem_alloc<1>(slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 1 && ptx::elect_one()) {
    const uint32_t idesc = ptx::idesc_tf32(128, n, 0, 0);
    const uint64_t bd = ptx::sdesc(ptx::smem_u32(smem), 16, 512, ptx::kLayoutSW64);
    const uint32_t a_t = tmem + 448;
    long long t0 = clock64();
    if (mode == 5 || mode == 6 || mode == 7 || mode == 8) {
      // the direct convolution's per-tile chain: 4 stages x 2 K-steps x 3 MMAs
      // (A_lo B_hi, A_hi B_lo, A_hi B_hi; B stages 6 KiB apart, hi / lo 24 KiB
      // apart), D alternating between two accumulators per tile, first MMA of a
      // tile not accumulating, then a commit per tile (mode 6: two)
      for (int r = 0, t = 0; r < reps; r += 24, ++t) {
        const uint32_t d = tmem + (t & 1) * n;
        for (int st = 0; st < 4; ++st)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t bH = bd + ((st * 6144) >> 4) + 2 * ks, bL = bH + (24576 >> 4);
            ptx::mma_tf32_tmem_a<1>(d, a_t + 16 + 8 * ks, bH, idesc, (st | ks) ? 1u : 0u);
            ptx::mma_tf32_tmem_a<1>(d, a_t + 8 * ks, bL, idesc, 1u);
            ptx::mma_tf32_tmem_a<1>(d, a_t + 8 * ks, bH, idesc, 1u);
          }
        if (mode >= 6) ptx::mma_commit<1>(bar);  // a commit per tile (phase flips unobserved: timing only)
      }
    } else {
    for (int r = 0; r < reps; r += 4) {
      ptx::mma_tf32_tmem_a<1>(tmem, a_t, bd, idesc, 1u);
      ptx::mma_tf32_tmem_a<1>(tmem, a_t + 8, bd + 2, idesc, 1u);
      ptx::mma_tf32_tmem_a<1>(tmem, a_t + 16, bd, idesc, 1u);
      ptx::mma_tf32_tmem_a<1>(tmem, a_t + 24, bd + 2, idesc, 1u);
    }
    }
    uint64_t* fin = bar + 4;
    ptx::mbar_init(fin, 1);
    ptx::fence_mbarrier_init();
    ptx::mma_commit<1>(fin);
    ptx::mbar_wait(fin, 0);
    long long t1 = clock64();
    *done = 1;
    if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
  } else if (((mode == 7 || mode == 9) && (warp & 3) == 1 && warp != 1) || (mode == 8 && (warp & 3) == 0 && warp != 0)) {
    // issue-slot competition: FFMA chains on the MMA warp's SMSP (mode 7: warps
    // 5, 9, 13 share SMSP 1 with warp 1) or on another SMSP (mode 8: 4, 8, 12)
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    unsigned long long ops = 0;
    while (!*done) {
#pragma unroll 16
      for (int i = 0; i < 256; ++i) {
        a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 1.0001f, 0.5f);
        a2 = fmaf(a2, 1.0001f, 0.5f); a3 = fmaf(a3, 1.0001f, 0.5f);
      }
      ++ops;
    }
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (warp == 5 || warp == 4)) out[1] = ops + (a0 + a1 + a2 + a3 == 0.f);
  } else if (warp >= 4 && mode >= 1 && mode <= 4) {
    const uint32_t row = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 256;
    uint32_t v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = j;
    unsigned long long ops = 0;
    while (!*done) {
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        if (mode == 1) {
          ptx::tmem_st_32x32b_x32(row + c, v);
          ptx::tmem_st_wait();
        } else if (mode == 4) {  // stores into the columns the MMAs read as A (timing only: racy values)
          ptx::tmem_st_32x32b_x32(row + 192, v);
          ptx::tmem_st_wait();
        } else if (mode == 3) {  // shared-memory reads (16 B per lane, 4 per round) from a region B does not use
          const uint32_t base = ptx::smem_u32(smem) + 32768 + (((warp & 3) * 32 + (threadIdx.x & 31)) * 16) + c * 64;
          uint4 a = ptx::lds128(base), b = ptx::lds128(base + 2048), e = ptx::lds128(base + 4096), f = ptx::lds128(base + 6144);
          v[0] += a.x + b.y + e.z + f.w;
        } else {
          uint32_t r[16];
          ptx::tmem_ld_32x32b_x16(row + c, r);
          ptx::tmem_ld_wait();
          v[0] += r[0];
        }
        ++ops;
      }
    }
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && warp == 4) out[1] = ops + (v[0] == 12345u);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem, 512);
  }
}

extern "C" int run_cont(int n, int reps, int mode, unsigned long long* mma_cycles, unsigned long long* side_ops) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  const int smem = 64 * 1024 + 2048;
  cudaFuncSetAttribute(k_cont, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_cont<<<148, 256, smem>>>(n, reps, mode, d);
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  *mma_cycles = h[0];
  *side_ops = h[1];
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
