// Does a same-device D2D cudaMemcpyAsync need SMs?  A spinner holds every SM
// for 3 ms (mode "smem": one 128-thread CTA per SM with ~200 KB of shared
// memory -- thread slots and registers left free; mode "threads": two
// 1024-thread CTAs per SM -- every thread slot taken, as the persistent GEMM
// takes every register); a 256 MiB device-to-device copy is enqueued on a
// second stream.  If the copy runs on copy engines it completes while the
// spinner runs; if it needs SMs it waits for them.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin(unsigned long long ns) {
  extern __shared__ char smem[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); smem[threadIdx.x] = (char)t; } while (t - t0 < ns);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t bytes = 256ull << 20;
  void *a, *b, *h;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMallocHost(&h, bytes);
  cudaMemset(a, 1, bytes);
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, k0, k1; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&k0); cudaEventCreate(&k1);
  const char* names[4] = {"D2D vs smem spinner", "D2H pinned vs smem spinner", "D2D alone", "D2D vs thread spinner"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(k0, s1);
      if (mode < 2) spin<<<sms, 128, 200 * 1024, s1>>>(3000000ull);
      if (mode == 3) spin<<<2 * sms, 1024, 1024, s1>>>(3000000ull);
      cudaEventRecord(k1, s1);
      cudaEventRecord(e0, s2);
      if (mode == 3) { unsigned long long t0 = 0; (void)t0; }
      cudaError_t err = cudaMemcpyAsync(mode == 1 ? h : b, a, bytes, mode == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s2);
      cudaEventRecord(e1, s2);
      cudaDeviceSynchronize();
      float tc = 0, tk = 0;
      cudaEventElapsedTime(&tc, e0, e1); cudaEventElapsedTime(&tk, k0, k1);
      printf("%s err=%s: copy %.3f ms (%.0f GB/s), spinner %.3f ms\n", names[mode], cudaGetErrorString(err), tc,
             bytes / (tc * 1e-3) / 1e9, tk);
    }
  }
  return 0;
}
