// tc_gemm.cu -- 3xTF32 split-operand sgemm on the sm_100a tensor cores.
//
// Computes C = alpha*A*B + beta*C in fp32-faithful accuracy:
// every fp32 operand x is split as x = hi + lo with hi = x truncated to TF32
// (the tensor core itself ignores the low 13 mantissa bits of a raw fp32
// operand in kind::tf32 -- probed -- so the raw TMA tile serves as hi) and
// lo = rna_tf32(x - hi) (exact subtraction, one rounding), and
//     A*B ~= A_lo*B_hi + A_hi*B_lo + A_hi*B_hi        (lo*lo dropped)
// accumulated in fp32.  The tensor core accumulates with round-toward-zero
// (probed), so partial sums over K_c = 128 live in TMEM and are promoted into
// round-to-nearest fp32 register accumulators ("K_c promotion", K_c = 128); see
// DESIGN.md "3xTF32 accuracy".
//
// Structure (the paper's GPU gemm optimisations, PAPER.md:69-71, 780, 830-831,
// mapped to Blackwell): two-level tiling = persistent cluster tiles (tiling map
// i0 = floor(i/BM), i1 = i % BM) x K-blocks of 32;
// "data movement between global, shared and register memory" = TMA into a
// multi-stage shared-memory ring + TMEM partials + register accumulators;
// "array packing" = the in-smem lo split; "synchronization primitives" =
// mbarrier full/empty rings; "separation of full and partial tiles" = TMA
// zero-fill for loads plus an explicit full-tile (unpredicated vector) /
// partial-tile (predicated) epilogue that fuses alpha/beta.
//
// Warp roles (512 threads = 4 warpgroups, 1 CTA per SM, persistent):
//   WG0 warp 0  TMA producer (one lane): A box 128x32 (K-major, SW128),
//               B boxes 32x32 (MN-major, SW128 with 32-B atoms) -> raw ring.
//       warp 1  MMA issuer (one lane, leader CTA only): 3 tcgen05.mma per K=8
//               step into one of two TMEM partial buffers (ping-pong per K_c).
//       warp 2  TMEM allocator.
//   WG1         split: raw tile -> lo tile (same swizzled layout, so the MMA
//               descriptors for lo differ from hi only in the start address).
//   WG2, WG3    promotion + epilogue: drain each finished TMEM partial into
//               fp32 registers (RN adds), then alpha/beta and store C.  Warp w
//               owns TMEM lanes 32*(w%4).. (rows) and column half (w-8)/4.
// CG == 2 runs a CTA pair (cta_group::2): tile 256 x (2*BN_CTA), A split along
// M and B along N between the two CTAs' shared memories; CTA 0 issues MMAs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "ptx.cuh"
#include "tm_internal.h"

namespace tmk {

constexpr int kBK = 32;            // K elements per stage (= one 128-byte swizzle row)
constexpr int kBMCta = 128;        // A rows per CTA
constexpr int kThreads = 512;
constexpr int kSplitThreads = 128;
constexpr int kEpiWarps = 8;
constexpr int kKcBlocksDefault = 4;   // K_c = 4 * 32 = 128: RZ partial length before RN promotion
constexpr int kGroupMDefault = 8;     // raster: tile-rows per group (L2 reuse)

template <int BN_CTA>
struct StageCfg;
template <>
struct StageCfg<128> { static constexpr int kRaw = 4, kLo = 2; };
template <>
struct StageCfg<64> { static constexpr int kRaw = 5, kLo = 3; };
template <>
struct StageCfg<32> { static constexpr int kRaw = 6, kLo = 3; };

template <int CG, int BN_CTA, bool SPLIT3>
struct TcCfg {
  static constexpr int kRaw = StageCfg<BN_CTA>::kRaw;
  static constexpr int kLo = StageCfg<BN_CTA>::kLo;  // ready/empty_lo ring depth (no lo smem if !SPLIT3)
  static constexpr int kABytes = kBMCta * kBK * 4;   // 16 KiB
  static constexpr int kBBytes = kBK * BN_CTA * 4;   // BN_CTA/32 boxes of 4 KiB
  static constexpr int kMmaM = kBMCta * CG;
  static constexpr int kMmaN = BN_CTA * CG;
  static constexpr int kTileM = kMmaM;
  static constexpr int kTileN = kMmaN;
  static constexpr int kCols = kMmaN / 2;            // columns per promotion warp
  static constexpr int kTmemCols = (2 * kMmaN <= 32) ? 32 : (2 * kMmaN <= 64) ? 64 : (2 * kMmaN <= 128) ? 128 : (2 * kMmaN <= 256) ? 256 : 512;
  static constexpr int kRawBytes = kRaw * (kABytes + kBBytes);
  static constexpr int kLoBytes = SPLIT3 ? kLo * (kABytes + kBBytes) : 0;
  static constexpr int kNumBars = 2 * kRaw + 2 * kLo + 4;
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kRawBytes + kLoBytes + kNumBars * 8 + 16;
};

struct TcParams {
  int m, n, k;
  int tiles_m, tiles_n, num_tiles, kblocks;
  int kc_blocks;  // K-blocks per TMEM partial (K_c / 32)
  int group_m;    // raster group height in tiles
  float alpha, beta;
  float* C;
  long long ldc;
};

// lo part of the 3xTF32 split of one fp32 value x (bit pattern):
//   hi = x with the low 13 mantissa bits cleared (what kind::tf32 reads from a
//        raw fp32 operand, probed: tests/test_probes.py),
//   d  = x - hi, exact in fp32,
//   lo = d rounded to TF32, round-to-nearest ties-away on the magnitude:
//        (bits(d) + 0x1000) & ~0x1FFF  (integer form of cvt.rna.tf32.f32 for
//        finite d; the carry into the exponent is the correct rounding).
__device__ __forceinline__ uint32_t tf32_lo_bits(uint32_t x) {
  const float hi = __uint_as_float(x & 0xFFFFE000u);
  const float d = __fsub_rn(__uint_as_float(x), hi);
  return (__float_as_uint(d) + 0x1000u) & 0xFFFFE000u;
}
__device__ __forceinline__ uint4 tf32_lo4(uint4 v) {
  return make_uint4(tf32_lo_bits(v.x), tf32_lo_bits(v.y), tf32_lo_bits(v.z), tf32_lo_bits(v.w));
}

// Split one smem tile of BYTES (raw -> lo, same offsets, so the same swizzled
// layout) with 128 threads, 8 loads in flight per thread.
template <int BYTES>
__device__ __forceinline__ void split_tile(uint32_t src, uint32_t dst, int st) {
  constexpr int kIters = BYTES / 16 / kSplitThreads;
  constexpr int kBatch = kIters < 8 ? kIters : 8;
#pragma unroll
  for (int b = 0; b < kIters; b += kBatch) {
    uint4 v[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) v[i] = ptx::lds128(src + ((b + i) * kSplitThreads + st) * 16);
#pragma unroll
    for (int i = 0; i < kBatch; ++i) ptx::sts128(dst + ((b + i) * kSplitThreads + st) * 16, tf32_lo4(v[i]));
  }
}

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group_m, int& tm_, int& tn_) {
  const int per_group = group_m * tiles_n;
  const int g = t / per_group;
  const int first_m = g * group_m;
  const int gsize = min(tiles_m - first_m, group_m);
  const int r = t - g * per_group;
  tm_ = first_m + r % gsize;
  tn_ = r / gsize;
}

// ------------------------------------------------------------------ epilogue
// Full tile: all KCOLS columns of this thread's row are inside C:
// unpredicated 16-byte vector accesses (ldc % 4 == 0 and C 16-B aligned are
// preconditions of this path).  Partial tile: row/column predicates, nothing
// outside m x n is touched.
template <int KCOLS>
__device__ __forceinline__ void epi_store(float* __restrict__ crow, const float (&acc)[KCOLS], bool full_row,
                                          int ncols, float alpha, float beta) {
  if (full_row) {
    float4* c4 = reinterpret_cast<float4*>(crow);
    if (beta == 0.0f) {
#pragma unroll
      for (int q = 0; q < KCOLS / 4; ++q)
        c4[q] = make_float4(alpha * acc[4 * q], alpha * acc[4 * q + 1], alpha * acc[4 * q + 2], alpha * acc[4 * q + 3]);
    } else {
#pragma unroll
      for (int q0 = 0; q0 < KCOLS / 4; q0 += 4) {
        float4 c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = c4[q0 + q];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = 4 * (q0 + q);
          c4[q0 + q] = make_float4(fmaf(alpha, acc[j], beta * c[q].x), fmaf(alpha, acc[j + 1], beta * c[q].y),
                                   fmaf(alpha, acc[j + 2], beta * c[q].z), fmaf(alpha, acc[j + 3], beta * c[q].w));
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < KCOLS; ++j) {
      if (j < ncols) crow[j] = (beta == 0.0f) ? alpha * acc[j] : fmaf(alpha, acc[j], beta * crow[j]);
    }
  }
}

template <int CG, int BN_CTA, bool SPLIT3>
__global__ void __launch_bounds__(kThreads, 1)
    k_sgemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
  using Cfg = TcCfg<CG, BN_CTA, SPLIT3>;
  constexpr int RAW = Cfg::kRaw, LO = Cfg::kLo, KCOLS = Cfg::kCols;

  extern __shared__ uint8_t smem_raw_[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_) + 1023) & ~uintptr_t(1023));
  uint8_t* rawA = smem;
  uint8_t* rawB = rawA + RAW * Cfg::kABytes;
  uint8_t* loA = rawB + RAW * Cfg::kBBytes;
  uint8_t* loB = loA + (SPLIT3 ? LO * Cfg::kABytes : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kRawBytes + Cfg::kLoBytes);
  uint64_t* full = bars;                   // [RAW] TMA landed (local)
  uint64_t* empty_raw = full + RAW;        // [RAW] MMA done with raw stage (commit, multicast)
  uint64_t* ready = empty_raw + RAW;       // [LO]  split done in all CTAs (leader)
  uint64_t* empty_lo = ready + LO;         // [LO]  MMA done with lo stage (commit, multicast)
  uint64_t* part_full = empty_lo + LO;     // [2]   TMEM partial complete (commit, multicast)
  uint64_t* part_empty = part_full + 2;    // [2]   partial drained by all promotion warps (leader)
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(part_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? ptx::cluster_ctarank() : 0;
  const int cluster_id = blockIdx.x / CG;
  const int num_clusters = gridDim.x / CG;

  if (threadIdx.x == 0) {
    for (int i = 0; i < RAW; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty_raw[i], 1);
    }
    for (int i = 0; i < LO; ++i) {
      ptx::mbar_init(&ready[i], (kSplitThreads / 32) * CG);
      ptx::mbar_init(&empty_lo[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&part_full[i], 1);
      ptx::mbar_init(&part_empty[i], kEpiWarps * CG);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 2) ptx::tmem_alloc<CG>(tmem_base_slot, Cfg::kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp < 4) {
    ptx::setmaxnreg_dec<80>();
    if (warp == 0) {
      // ---------------------------------------------------------- producer
      if (ptx::elect_one()) {
        int s = 0;
        uint32_t ph = 0;
        for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
          int tmi, tni;
          tile_coords(t, p.tiles_m, p.tiles_n, p.group_m, tmi, tni);
          const int row0 = tmi * Cfg::kTileM + static_cast<int>(rank) * kBMCta;
          const int col0 = tni * Cfg::kTileN + static_cast<int>(rank) * BN_CTA;
          for (int kb = 0; kb < p.kblocks; ++kb) {
            ptx::mbar_wait(&empty_raw[s], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&full[s], Cfg::kABytes + Cfg::kBBytes);
            ptx::tma_load_2d(rawA + s * Cfg::kABytes, &tmA, &full[s], kb * kBK, row0);
#pragma unroll
            for (int j = 0; j < BN_CTA / 32; ++j)
              ptx::tma_load_2d(rawB + s * Cfg::kBBytes + j * 4096, &tmB, &full[s], col0 + 32 * j, kb * kBK);
            if (++s == RAW) { s = 0; ph ^= 1; }
          }
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      if (rank == 0 && ptx::elect_one()) {
        constexpr uint32_t idesc = ptx::idesc_tf32(Cfg::kMmaM, Cfg::kMmaN, /*A MN-major*/ 0, /*B MN-major*/ 1);
        const uint32_t rawA_s = ptx::smem_u32(rawA), rawB_s = ptx::smem_u32(rawB);
        const uint32_t loA_s = ptx::smem_u32(loA), loB_s = ptx::smem_u32(loB);
        int s = 0, sl = 0, pb = 0;
        uint32_t ph = 0, phl = 0, pph = 0;
        for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
          for (int kb0 = 0; kb0 < p.kblocks; kb0 += p.kc_blocks) {
            const int kb1 = min(kb0 + p.kc_blocks, p.kblocks);
            ptx::mbar_wait_cluster(&part_empty[pb], pph ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + static_cast<uint32_t>(pb * Cfg::kMmaN);
            for (int kb = kb0; kb < kb1; ++kb) {
              ptx::mbar_wait_cluster(&ready[sl], phl);
              ptx::tc_fence_after();
#pragma unroll
              for (int ks = 0; ks < kBK / 8; ++ks) {
                // A: K-major SW128, K step of 8 tf32 = 32 B inside the swizzle row.
                // B: MN-major SW128_BASE32B, K step of 8 rows = 1024 B (two 512-B
                //    atoms, SBO); 32-column atoms are 4096 B apart (LBO).
                const uint64_t aH = ptx::sdesc(rawA_s + s * Cfg::kABytes + ks * 32, 16, 1024, ptx::kLayoutSW128);
                const uint64_t bH =
                    ptx::sdesc(rawB_s + s * Cfg::kBBytes + ks * 1024, 4096, 512, ptx::kLayoutSW128Base32B);
                const uint32_t acc = (kb != kb0 || ks != 0) ? 1u : 0u;  // fresh partial per K_c chunk
                if constexpr (SPLIT3) {
                  const uint64_t aL = ptx::sdesc(loA_s + sl * Cfg::kABytes + ks * 32, 16, 1024, ptx::kLayoutSW128);
                  const uint64_t bL =
                      ptx::sdesc(loB_s + sl * Cfg::kBBytes + ks * 1024, 4096, 512, ptx::kLayoutSW128Base32B);
                  ptx::mma_tf32<CG>(d, aL, bH, idesc, acc);
                  ptx::mma_tf32<CG>(d, aH, bL, idesc, 1u);
                  ptx::mma_tf32<CG>(d, aH, bH, idesc, 1u);
                } else {
                  ptx::mma_tf32<CG>(d, aH, bH, idesc, acc);
                }
              }
              ptx::mma_commit<CG>(&empty_raw[s]);
              ptx::mma_commit<CG>(&empty_lo[sl]);  // also paces the ready ring when !SPLIT3
              if (++s == RAW) { s = 0; ph ^= 1; }
              if (++sl == LO) { sl = 0; phl ^= 1; }
            }
            ptx::mma_commit<CG>(&part_full[pb]);
            if (++pb == 2) { pb = 0; pph ^= 1; }
          }
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ split
    ptx::setmaxnreg_dec<80>();
    const int st = threadIdx.x - 128;
    const uint32_t rawA_s = ptx::smem_u32(rawA), rawB_s = ptx::smem_u32(rawB);
    const uint32_t loA_s = ptx::smem_u32(loA), loB_s = ptx::smem_u32(loB);
    int s = 0, sl = 0;
    uint32_t ph = 0, phl = 0;
    for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
      for (int kb = 0; kb < p.kblocks; ++kb) {
        ptx::mbar_wait(&full[s], ph);
        // The ready ring must not run more than LO stages ahead of the MMA
        // (an mbarrier phase may not complete twice before it is observed).
        ptx::mbar_wait(&empty_lo[sl], phl ^ 1);
        if constexpr (SPLIT3) {
          split_tile<Cfg::kABytes>(rawA_s + s * Cfg::kABytes, loA_s + sl * Cfg::kABytes, st);
          split_tile<Cfg::kBBytes>(rawB_s + s * Cfg::kBBytes, loB_s + sl * Cfg::kBBytes, st);
          ptx::fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) ptx::mbar_arrive_cluster(&ready[sl], 0);
          else ptx::mbar_arrive(&ready[sl]);
        }
        if (++s == RAW) { s = 0; ph ^= 1; }
        if (++sl == LO) { sl = 0; phl ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ promotion + epilogue
    ptx::setmaxnreg_inc<176>();
    const int q = warp & 3;             // TMEM lane quarter (rows 32q..32q+31 of this CTA)
    const int h = (warp - 8) >> 2;      // column half
    int pb = 0;
    uint32_t pph = 0;
    for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
      int tmi, tni;
      tile_coords(t, p.tiles_m, p.tiles_n, p.group_m, tmi, tni);
      float acc[KCOLS];
#pragma unroll
      for (int j = 0; j < KCOLS; ++j) acc[j] = 0.0f;
      for (int kb0 = 0; kb0 < p.kblocks; kb0 += p.kc_blocks) {
        ptx::mbar_wait(&part_full[pb], pph);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                               static_cast<uint32_t>(pb * Cfg::kMmaN + h * KCOLS);
#pragma unroll
        for (int c = 0; c < KCOLS; c += 16) {
          uint32_t r[16];
          ptx::tmem_ld_32x32b_x16(taddr + c, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[c + j] += __uint_as_float(r[j]);  // RN promotion
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) ptx::mbar_arrive_cluster(&part_empty[pb], 0);
          else ptx::mbar_arrive(&part_empty[pb]);
        }
        if (++pb == 2) { pb = 0; pph ^= 1; }
      }
      const int row = tmi * Cfg::kTileM + static_cast<int>(rank) * kBMCta + q * 32 + lane;
      const int col0 = tni * Cfg::kTileN + h * KCOLS;
      if (row < p.m && col0 < p.n) {
        const bool full_row = (col0 + KCOLS <= p.n);
        epi_store<KCOLS>(p.C + static_cast<long long>(row) * p.ldc + col0, acc, full_row, p.n - col0, p.alpha,
                         p.beta);
      }
    }
  }

  // ---------------------------------------------------------------- teardown
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, Cfg::kTmemCols);
  }
}

// ------------------------------------------------------------------ host side
namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D fp32 row-major tensor (rows x cols, leading dimension ld elements),
// box = box_cols x box_rows, 128-byte swizzle span, OOB elements read as zero.
bool encode_2d(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_cols,
               uint32_t box_rows, CUtensorMapSwizzle swizzle) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int CG, int BN_CTA, bool SPLIT3>
tm_status launch_cfg(const GemmArgs& a, int num_sms, cudaStream_t stream) {
  using Cfg = TcCfg<CG, BN_CTA, SPLIT3>;
  auto kern = k_sgemm_tc<CG, BN_CTA, SPLIT3>;
  static bool attr_set = false;  // per instantiation; attribute is per-function, process-wide
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes) != cudaSuccess)
      return TM_ERR_CUDA;
    attr_set = true;
  }
  CUtensorMap tmA, tmB;
  // A: m x k, box 32 (k) x 128 (rows).  B: k x n, box 32 (n) x 32 (k rows).
  if (!encode_2d(&tmA, a.A, a.m, a.k, a.lda, kBK, kBMCta, CU_TENSOR_MAP_SWIZZLE_128B)) return TM_ERR_INTERNAL;
  if (!encode_2d(&tmB, a.B, a.k, a.n, a.ldb, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return TM_ERR_INTERNAL;
  TcParams p;
  p.m = static_cast<int>(a.m);
  p.n = static_cast<int>(a.n);
  p.k = static_cast<int>(a.k);
  p.tiles_m = static_cast<int>((a.m + Cfg::kTileM - 1) / Cfg::kTileM);
  p.tiles_n = static_cast<int>((a.n + Cfg::kTileN - 1) / Cfg::kTileN);
  p.num_tiles = p.tiles_m * p.tiles_n;
  p.kblocks = static_cast<int>((a.k + kBK - 1) / kBK);
  p.kc_blocks = kKcBlocksDefault;
  p.group_m = kGroupMDefault;
  if (const char* e = std::getenv("TM_KC_BLOCKS")) p.kc_blocks = std::max(1, std::atoi(e));  // tuning knob
  if (const char* e = std::getenv("TM_GROUP_M")) p.group_m = std::max(1, std::atoi(e));     // tuning knob
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.C = a.C;
  p.ldc = a.ldc;
  const int max_clusters = num_sms / CG;
  const int clusters = p.num_tiles < max_clusters ? p.num_tiles : max_clusters;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * CG, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, tmA, tmB, p) != cudaSuccess) return TM_ERR_CUDA;
  return TM_OK;
}

template <bool SPLIT3>
tm_status launch_split(const GemmArgs& a, int cg, int bn, int num_sms, cudaStream_t s) {
  if (cg == 2) {
    if (bn == 128) return launch_cfg<2, 128, SPLIT3>(a, num_sms, s);
    if (bn == 64) return launch_cfg<2, 64, SPLIT3>(a, num_sms, s);
    if (bn == 32) return launch_cfg<2, 32, SPLIT3>(a, num_sms, s);
  } else if (cg == 1) {
    if (bn == 128) return launch_cfg<1, 128, SPLIT3>(a, num_sms, s);
    if (bn == 64) return launch_cfg<1, 64, SPLIT3>(a, num_sms, s);
    if (bn == 32) return launch_cfg<1, 32, SPLIT3>(a, num_sms, s);
  }
  return TM_ERR_INVALID_VALUE;
}

}  // namespace

tm_status launch_tc(const GemmArgs& a, const TcChoice& c, int num_sms, cudaStream_t stream) {
  if (a.m > INT32_MAX / 2 || a.n > INT32_MAX / 2 || a.k > INT32_MAX / 2) return TM_ERR_INVALID_VALUE;
  return c.split3 ? launch_split<true>(a, c.cg, c.bn_cta, num_sms, stream)
                  : launch_split<false>(a, c.cg, c.bn_cta, num_sms, stream);
}

}  // namespace tmk
