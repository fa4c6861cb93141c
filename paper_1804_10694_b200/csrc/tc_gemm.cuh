// tc_gemm.cuh -- 3xTF32 split-operand sgemm on the sm_100a tensor cores
// (kernel + host launch templates; instantiated per operand layout in
// tc_gemm_{nn,nt,tn,tt}.cu so the four variants compile in parallel).
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
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"
#include "tm_internal.h"

// Mutation testing of the tests (tests/test_product_mutants.py): a library
// built with -DTM_MUTATE=n breaks exactly one guard on purpose and the named
// test must then fail ("Mutation tests").  The shipped
// build has TM_MUTATE == 0 and every TM_MUT(n) is the constant false.
//   1  the epilogue's partial-tile predicate is ignored (every 4-column group
//      is stored as a full vector): the guard-band test must fail
//   2  the B_lo split term is dropped (stored as zero): the 1e-5 parity tests must fail
#ifndef TM_MUTATE
#define TM_MUTATE 0
#endif
#define TM_MUT(n) (TM_MUTATE == (n))

namespace tmk {

constexpr int kBK = 32;            // K elements per stage (= one 128-byte swizzle row)
constexpr int kBMCta = 128;        // A rows per CTA
constexpr int kThreads = 512;
constexpr int kSplitThreads = 128;
constexpr int kEpiWarps = 8;
constexpr int kProducers = 3;      // TMA-issuing warps (0, 2, 3)
constexpr int kEpiStride = 20;     // floats per staged row (16 data + 4 pad: 16-B aligned, few bank conflicts)
constexpr int kKcBlocksDefault = 4;   // K_c = 4 * 32 = 128: RZ partial length before RN promotion
// Raster: tile-rows per group (L2 reuse).  A wave of 74 concurrent 256x256
// tiles touches GROUP_M A panels and 74/GROUP_M B panels, minimal near
// sqrt(74): 8 cuts C5's DRAM reads 22.0 -> 18.8 GB per launch at the same
// throughput as 16 (scripts/r02/groupm.sh).
constexpr int kGroupMDefault = 8;

// Precision variants of the tensor-core path (template parameter PREC):
//   kPrecTf32x1  one kind::tf32 MMA per K step on the raw operands (fast, ~2e-3);
//   kPrecTf32x3  x = hi + lo split, A_lo B_hi + A_hi B_lo + A_hi B_hi (the default);
//   kPrecBf16x9  x = b0 + b1 + b2, three bf16 pieces that represent every fp32
//                exactly (8 + 8 + 8 significant bits), all nine products
//                sum_ij a_i b_j on kind::f16 MMAs (each product exact in fp32).
constexpr int kPrecTf32x1 = 0, kPrecTf32x3 = 1, kPrecBf16x9 = 2;

// Stage ring sizes from a shared-memory budget.  With A_lo in TMEM (kAlo: K-major
// A and room for at least two A_lo stages beyond the two partial accumulators)
// the lo ring holds only B_lo in shared memory and A_lo in TMEM columns, so it
// is made as deep as TMEM allows (<= 8; also 8 for 1xTF32): for skinny tiles a stage carries only
// a few short MMAs, and a 2-deep split -> MMA -> commit round trip would bound
// the rate.  Otherwise two lo stages; as many raw (TMA) stages as fit, <= 12.
// BF16x9: the "lo" ring holds the split stage -- three bf16 planes of A (128
// rows) and of B (BN_CTA rows), each K-major with 64-byte rows (32 k).
template <int CG, int BN_CTA, int PREC, int BK = 32, bool TA = false>
struct TcCfg {
  static constexpr bool SPLIT3 = PREC == kPrecTf32x3;
  static constexpr bool BF16 = PREC == kPrecBf16x9;
  static constexpr int kABytes = kBMCta * BK * 4;    // 16 KiB (BK 32) / 8 KiB (BK 16)
  static constexpr int kBBytes = BK * BN_CTA * 4;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kPlaneA = kBMCta * BK * 2;    // one bf16 plane of A (BF16x9)
  static constexpr int kPlaneB = BN_CTA * BK * 2;
  static constexpr int kSplitStage = 3 * (kPlaneA + kPlaneB);
  static constexpr int kMmaM = kBMCta * CG;
  static constexpr int kMmaN = BN_CTA * CG;
  static constexpr bool kAlo = SPLIT3 && !TA && (2 * kMmaN + 2 * BK <= 512);
  static constexpr int kLoFit = (200 * 1024 - 6 * kStage) / kBBytes;  // keep >= 6 raw stages
  static constexpr int kLoTmem0 = kAlo ? (512 - 2 * kMmaN) / BK : 2;
  static constexpr int kLoTmem = kLoTmem0 < kLoFit ? kLoTmem0 : (kLoFit < 2 ? 2 : kLoFit);
  // ready/empty_lo ring depth (only pacing barriers, no storage, for 1xTF32)
  static constexpr int kLo = PREC == kPrecTf32x1 ? 8 : kAlo ? (kLoTmem < 8 ? kLoTmem : 8) : 2;
  static constexpr int kLoBytes = BF16 ? kLo * kSplitStage : SPLIT3 ? kLo * (kAlo ? kBBytes : kStage) : 0;
  static constexpr int kRawFit = (200 * 1024 - kLoBytes) / kStage;
  static constexpr int kRaw = kRawFit < 12 ? kRawFit : 12;
  static constexpr int kTileM = kMmaM;
  static constexpr int kTileN = kMmaN;
  static constexpr int kCols = kMmaN / 2;            // columns per promotion warp
  static constexpr int kRawBytes = kRaw * kStage;
  static constexpr int kNumBars = 2 * kRaw + 2 * kLo + 4;
  static constexpr int kEpiStageBytes = kEpiWarps * 32 * kEpiStride * 4;  // transpose staging
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kRawBytes + kLoBytes + kEpiStageBytes + kNumBars * 8 + 16;
  static_assert(kRaw >= 3, "ring too shallow");
  static_assert(!BF16 || BK == 32, "BF16x9: 32-k stages");
  static_assert(kSmemBytes <= 227 * 1024, "shared memory");
};

struct TcParams {
  const float* A;  // raw pointers for L2 prefetch (the TMA maps carry the same tensors)
  long long lda;
  int m, n, k;
  int tiles_m, tiles_n, num_tiles, kblocks;
  int kc_blocks;  // K-blocks per TMEM partial (K_c / 32)
  int group_m;    // raster group height in tiles
  // stream-K: the iteration space of the first
  // sk_tiles tiles (sk_tiles x kblocks) is cut into equal contiguous ranges, one
  // per cluster; tiles split between clusters are reduced in a fixed order
  // through a workspace (deterministic).  Hybrid schedule: sk_tiles < num_tiles
  // -- every cluster first works its stream-K share, then the remaining tiles
  // whole, data-parallel (tile sk_tiles + cluster + j * clusters), so the
  // fixed-order reductions overlap whole tiles' streaming instead of forming the
  // kernel's tail.
  int streamk;
  int sk_tiles;            // tiles in the stream-K region (num_tiles: pure stream-K)
  long long iters;         // sk_tiles * kblocks
  float* ws;               // [clusters][CG][128][kMmaN] fp32 partials
  unsigned* flags;         // [clusters][CG][kEpiWarps] epoch flags
  unsigned epoch;          // this launch's flag value
  float alpha, beta;
  float* C;
  long long ldc;
  unsigned long long* trace;  // debug timeline [grid][kTraceSlots] (%globaltimer ns) or null
  unsigned* wave_ctr;         // data-parallel wave barrier counter (zeroed per launch) or null
  int full_waves;             // waves in which every cluster has a tile
  // fused distributed mode: B's K-chunk c (kchunk_blocks K-blocks) may be read
  // once kflags[c] >= kepoch (set by the transfer stream); null otherwise
  const unsigned* kflags;
  unsigned kepoch;
  int kchunk_blocks;
  // implicit-GEMM convolution (CONV kernels): GEMM row = output pixel
  // (b, y, x) of an Nb x Ho x Wo grid, K index = (ky*S + kx)*C + c.
  int cv_ho, cv_wo, cv_s, cv_c, cv_pad;
};

constexpr int kTraceSlots = 16;
__device__ __forceinline__ void trace_mark(const TcParams& p, int slot) {
  if (p.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * kTraceSlots + slot] = t;
  }
}

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
__device__ __forceinline__ void zero_tile(uint32_t dst, int st) {  // TM_MUTATE == 2 only
  for (int idx = st; idx < BYTES / 16; idx += kSplitThreads) ptx::sts128(dst + idx * 16, make_uint4(0u, 0u, 0u, 0u));
}

template <int BYTES>
__device__ __forceinline__ void split_tile(uint32_t src, uint32_t dst, int st) {
  constexpr int kChunks = BYTES / 16;
  constexpr int kIters = (kChunks + kSplitThreads - 1) / kSplitThreads;
  constexpr int kBatch = kIters < 8 ? kIters : 8;
  constexpr bool kRagged = kChunks % kSplitThreads != 0;  // tiles smaller than 128 x 16 B
#pragma unroll
  for (int b = 0; b < kIters; b += kBatch) {
    uint4 v[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int idx = (b + i) * kSplitThreads + st;
      if (!kRagged || idx < kChunks) v[i] = ptx::lds128(src + idx * 16);
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int idx = (b + i) * kSplitThreads + st;
      if (!kRagged || idx < kChunks) ptx::sts128(dst + idx * 16, tf32_lo4(v[i]));
    }
  }
}

// ---- BF16x9 split (kPrecBf16x9) ----
// x = b0 + b1 + b2 exactly: b0 = RN_bf16(x), b1 = RN_bf16(x - b0),
// b2 = RN_bf16(x - b0 - b1); both subtractions are exact in fp32 and the last
// remainder has at most 8 significant bits, so b2 is exact too (normal range).
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {  // lo -> bits 0..15
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ void split8_bf16(const float (&x)[8], uint4& p0, uint4& p1, uint4& p2) {
  uint32_t w0[4], w1[4], w2[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float a = x[2 * j], b = x[2 * j + 1];
    w0[j] = pack_bf16x2(a, b);
    const float ra = __fsub_rn(a, bf16_lo(w0[j])), rb = __fsub_rn(b, bf16_hi(w0[j]));
    w1[j] = pack_bf16x2(ra, rb);
    w2[j] = pack_bf16x2(__fsub_rn(ra, bf16_lo(w1[j])), __fsub_rn(rb, bf16_hi(w1[j])));
  }
  p0 = make_uint4(w0[0], w0[1], w0[2], w0[3]);
  p1 = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  p2 = make_uint4(w2[0], w2[1], w2[2], w2[3]);
}
// Row r of a raw fp32 stage -> the three bf16 planes of the split stage.
//   KMAJOR_SRC: the raw tile is K-major, TMA SWIZZLE_128B (row r = 128 B of 32 k,
//               16-B chunk c at c ^ (r % 8));
//   else        MN-major without swizzle, rows of `ld_src` floats per k
//               (element (k, r) at (k * ld_src + r) * 4).
// Each plane is K-major with 64-B rows (32 bf16), SWIZZLE_64B: row r at
// (r / 8) * 512 + (r % 8) * 64, 16-B chunk q at q ^ ((r / 2) % 4).
template <bool KMAJOR_SRC>
__device__ __forceinline__ void split_row_bf16(uint32_t src, int ld_src, int r, uint32_t plane0, uint32_t plane_bytes) {
  const uint32_t drow = plane0 + (r >> 3) * 512 + (r & 7) * 64;
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // k in [8q, 8q + 8)
    float x[8];
    if constexpr (KMAJOR_SRC) {
      const uint32_t row = src + r * 128;
      const uint4 v0 = ptx::lds128(row + (((2 * q) ^ (r & 7)) << 4));
      const uint4 v1 = ptx::lds128(row + (((2 * q + 1) ^ (r & 7)) << 4));
      x[0] = __uint_as_float(v0.x); x[1] = __uint_as_float(v0.y); x[2] = __uint_as_float(v0.z); x[3] = __uint_as_float(v0.w);
      x[4] = __uint_as_float(v1.x); x[5] = __uint_as_float(v1.y); x[6] = __uint_as_float(v1.z); x[7] = __uint_as_float(v1.w);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t w;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w) : "r"(src + ((8 * q + j) * ld_src + r) * 4));
        x[j] = __uint_as_float(w);
      }
    }
    uint4 p0, p1, p2;
    split8_bf16(x, p0, p1, p2);
    const uint32_t off = drow + ((q ^ ((r >> 1) & 3)) << 4);
    ptx::sts128(off, p0);
    ptx::sts128(off + plane_bytes, p1);
    ptx::sts128(off + 2 * plane_bytes, p2);
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

// Work units: (tile, K-block range).  Data-parallel: whole tiles c, c+C, ...
// Stream-K: cluster c owns iterations [c*I/C, (c+1)*I/C) of I = tiles x
// kblocks; its first unit may start inside a tile (a "partial" unit, written to
// the workspace), its last may end inside one (the tile's "finalizer", which
// adds the later clusters' partials in cluster order).
struct Unit {
  int tile, kb0, kb1;
  bool dp;  // a whole data-parallel tile (the wave barrier counts these)
};
struct UnitIter {
  long long it, end;  // stream-K cursor
  int next_tile;      // data-parallel cursor
};
__device__ __forceinline__ long long sk_start(long long iters, int c, int C) { return iters * c / C; }
__device__ __forceinline__ UnitIter units_begin(const TcParams& p, int cluster, int C) {
  UnitIter u;
  u.it = p.streamk ? sk_start(p.iters, cluster, C) : 0;
  u.end = p.streamk ? sk_start(p.iters, cluster + 1, C) : 0;
  u.next_tile = (p.streamk ? p.sk_tiles : 0) + cluster;
  return u;
}
__device__ __forceinline__ bool units_next(const TcParams& p, int C, UnitIter& s, Unit& u) {
  if (!p.streamk || s.it >= s.end) {  // data-parallel tiles (after the stream-K share, if any)
    if (s.next_tile >= p.num_tiles) return false;
    u.tile = s.next_tile;
    u.kb0 = 0;
    u.kb1 = p.kblocks;
    u.dp = true;
    s.next_tile += C;
    return true;
  }
  u.dp = false;
  u.tile = static_cast<int>(s.it / p.kblocks);
  u.kb0 = static_cast<int>(s.it - static_cast<long long>(u.tile) * p.kblocks);
  const long long left = s.end - s.it;
  u.kb1 = (left < p.kblocks - u.kb0) ? u.kb0 + static_cast<int>(left) : p.kblocks;
  s.it += u.kb1 - u.kb0;
  return true;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Spin until *p reaches a value (>= target, or == target when exact): the
// grid-wide waits of the wave barrier and the stream-K finalizer.  All
// clusters are co-resident (cooperative launch), so these complete unless a
// schedule bug leaves a producer without work; then trap after ~20 s instead
// of hanging the device.
static __device__ __forceinline__ void spin_until(const unsigned* p, unsigned target, bool exact, unsigned sleep_ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    const unsigned v = ld_acquire_gpu(p);
    if (exact ? v == target : v >= target) return;
    __nanosleep(sleep_ns);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) __trap();
  }
}

// Fused distributed mode: wait until B's K-chunk c has arrived (its flag,
// written by a stream memory operation after the chunk's transfer, reaches
// this call's epoch), then order the TMA (async-proxy) reads of that chunk
// after the acquire.  A transfer that never completes traps after ~20 s
// instead of hanging the device.
static __device__ __noinline__ void wait_chunk_flag(const unsigned* flag, unsigned epoch) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (static_cast<int>(ld_acquire_gpu(flag) - epoch) < 0) {
    __nanosleep(200);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) __trap();
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------------ epilogue
// C[row0 + r, col0 + j] = alpha*acc + beta*C for this warp's 32 rows x KCOLS
// columns, where lane r holds row r (the TMEM lane mapping).  Coalescing: each
// 16-column slab is transposed through a per-warp shared-memory stage so that
// every warp-wide access covers 8 rows x 64 contiguous bytes (8 L1 wavefronts)
// instead of 32 rows x 16 bytes.  Full/partial tile separation: a 4-column
// group entirely inside C uses one 16-byte vector access; groups crossing the
// right edge, and rows past m, are predicated element by element -- nothing
// outside m x n is read or written.  beta == 0 never reads C.
template <int KCOLS>
__device__ __forceinline__ void epi_store_lowreg(float* __restrict__ C, long long ldc, int m, int n, int row0, int col0,
                                          const float (&acc)[KCOLS], float alpha, float beta, float* stage,
                                          int lane) {
  constexpr int SWD = KCOLS < 16 ? KCOLS : 16;  // slab width (columns)
  constexpr int G = SWD / 4;                     // 16-byte groups per slab row
  constexpr int RPI = 32 / G;                    // rows covered by one warp-wide access
  constexpr int NI = 32 / RPI;                   // accesses per slab
#pragma unroll
  for (int c = 0; c < KCOLS; c += SWD) {
#pragma unroll
    for (int j = 0; j < SWD; j += 4)
      *reinterpret_cast<float4*>(stage + lane * kEpiStride + j) =
          make_float4(acc[c + j], acc[c + j + 1], acc[c + j + 2], acc[c + j + 3]);
    __syncwarp();
    const int cc = (lane % G) * 4;
    const int col = col0 + c + cc;
    const bool full_cols = TM_MUT(1) || col + 3 < n;
#pragma unroll
    for (int i0 = 0; i0 < NI; i0 += 2) {  // two row groups per round: 2 C loads in flight, low register use
      float4 v[2], cv[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = (i0 + i) * RPI + lane / G;
        v[i] = *reinterpret_cast<const float4*>(stage + r * kEpiStride + cc);
        cv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int row = row0 + r;
        if (beta != 0.0f && row < m) {
          const float* cp = C + static_cast<long long>(row) * ldc + col;
          if (full_cols) {
            cv[i] = *reinterpret_cast<const float4*>(cp);
          } else {
            if (col < n) cv[i].x = cp[0];
            if (col + 1 < n) cv[i].y = cp[1];
            if (col + 2 < n) cv[i].z = cp[2];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int row = row0 + (i0 + i) * RPI + lane / G;
        if (row >= m) continue;
        float4 o;
        if (beta == 0.0f) {
          o = make_float4(alpha * v[i].x, alpha * v[i].y, alpha * v[i].z, alpha * v[i].w);
        } else {
          o = make_float4(fmaf(alpha, v[i].x, beta * cv[i].x), fmaf(alpha, v[i].y, beta * cv[i].y),
                          fmaf(alpha, v[i].z, beta * cv[i].z), fmaf(alpha, v[i].w, beta * cv[i].w));
        }
        float* cp = C + static_cast<long long>(row) * ldc + col;
        if (full_cols) {
          *reinterpret_cast<float4*>(cp) = o;
        } else {
          if (col < n) cp[0] = o.x;
          if (col + 1 < n) cp[1] = o.y;
          if (col + 2 < n) cp[2] = o.z;
        }
      }
    }
    __syncwarp();
  }
}

template <int KCOLS>
__device__ __forceinline__ void epi_store(float* __restrict__ C, long long ldc, int m, int n, int row0, int col0,
                                          const float (&acc)[KCOLS], float alpha, float beta, float* stage,
                                          int lane) {
  constexpr int SWD = KCOLS < 16 ? KCOLS : 16;  // slab width (columns)
  constexpr int G = SWD / 4;                     // 16-byte groups per slab row
  constexpr int RPI = 32 / G;                    // rows covered by one warp-wide access
  constexpr int NI = 32 / RPI;                   // accesses per slab
  constexpr int NSLAB = KCOLS / SWD;
  // beta*C loads issued together: the epilogue is bound by the C-load round
  // trip (L2 or DRAM), so for KCOLS <= 64 all of a warp's loads go out at once
  // (SB slabs x RB row groups = KCOLS extra registers); KCOLS 128, whose 128
  // accumulator registers leave no room, keeps two loads in flight per slab.
  if constexpr (NSLAB > 4) {
    epi_store_lowreg<KCOLS>(C, ldc, m, n, row0, col0, acc, alpha, beta, stage, lane);
    return;
  }
  constexpr int SB = NSLAB <= 4 ? NSLAB : 1;
  constexpr int RB = NSLAB <= 4 ? NI : 2;
  const int cc = (lane % G) * 4;
#pragma unroll
  for (int c0 = 0; c0 < NSLAB; c0 += SB) {
#pragma unroll
    for (int i0 = 0; i0 < NI; i0 += RB) {
      float4 cv[SB][RB];
#pragma unroll
      for (int sb = 0; sb < SB; ++sb) {
        const int col = col0 + (c0 + sb) * SWD + cc;
        const bool full_cols = TM_MUT(1) || col + 3 < n;
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          cv[sb][i] = make_float4(0.f, 0.f, 0.f, 0.f);
          const int row = row0 + (i0 + i) * RPI + lane / G;
          if (beta != 0.0f && row < m) {
            const float* cp = C + static_cast<long long>(row) * ldc + col;
            if (full_cols) {
              cv[sb][i] = *reinterpret_cast<const float4*>(cp);
            } else {
              if (col < n) cv[sb][i].x = cp[0];
              if (col + 1 < n) cv[sb][i].y = cp[1];
              if (col + 2 < n) cv[sb][i].z = cp[2];
            }
          }
        }
      }
#pragma unroll
      for (int sb = 0; sb < SB; ++sb) {
        const int c = (c0 + sb) * SWD;
        if (i0 == 0) {  // stage this slab (lane = row) for row-group reads
#pragma unroll
          for (int j = 0; j < SWD; j += 4)
            *reinterpret_cast<float4*>(stage + lane * kEpiStride + j) =
                make_float4(acc[c + j], acc[c + j + 1], acc[c + j + 2], acc[c + j + 3]);
          __syncwarp();
        }
        const int col = col0 + c + cc;
        const bool full_cols = TM_MUT(1) || col + 3 < n;
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          const int r = (i0 + i) * RPI + lane / G;
          const int row = row0 + r;
          const float4 v = *reinterpret_cast<const float4*>(stage + r * kEpiStride + cc);
          if (row >= m) continue;
          float4 o;
          if (beta == 0.0f) {
            o = make_float4(alpha * v.x, alpha * v.y, alpha * v.z, alpha * v.w);
          } else {
            const float4 q = cv[sb][i];
            o = make_float4(fmaf(alpha, v.x, beta * q.x), fmaf(alpha, v.y, beta * q.y),
                            fmaf(alpha, v.z, beta * q.z), fmaf(alpha, v.w, beta * q.w));
          }
          float* cp = C + static_cast<long long>(row) * ldc + col;
          if (full_cols) {
            *reinterpret_cast<float4*>(cp) = o;
          } else {
            if (col < n) cp[0] = o.x;
            if (col + 1 < n) cp[1] = o.y;
            if (col + 2 < n) cp[2] = o.z;
          }
        }
        if (i0 + RB == NI) __syncwarp();  // slab done: the stage may be rewritten
      }
    }
  }
}

// TA / TB: op(A) = A^T (A stored k x m, M contiguous -> MN-major A operand) /
// op(B) = B^T (B stored n x k, K contiguous -> K-major B operand).
// BK: K elements per stage, 32 (128-B K-major rows, SWIZZLE_128B) or 16 (64-B
// rows, SWIZZLE_64B; K-major operands only).
// CONV: A is the implicit im2col matrix of an NHWC activation tensor, loaded
// with TMA im2col-mode copies (one filter tap x BK channels per stage).
template <int CG, int BN_CTA, int PREC, bool TA, bool TB, int BK = 32, bool CONV = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_sgemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
  using Cfg = TcCfg<CG, BN_CTA, PREC, BK, TA>;
  constexpr bool SPLIT3 = Cfg::SPLIT3;  // 3xTF32
  constexpr bool BF16 = Cfg::BF16;      // BF16x9
  static_assert(!BF16 || !CONV, "BF16x9: GEMM only");
  static_assert(BK == 32 || BK == 16, "BK");
  static_assert(BK == 32 || (!TA && TB), "64-B rows only for K-major operands");
  static_assert(TB || BN_CTA % 32 == 0, "MN-major B needs 32-column atoms");
  static_assert(!CONV || (!TA && TB), "conv: A = im2col (K-major), B = KRSC filters (K-major)");
  constexpr int RAW = Cfg::kRaw, LO = Cfg::kLo, KCOLS = Cfg::kCols;
  // A_lo staged in TMEM (written by the split warps with tcgen05.st, read by
  // the A_lo*B_hi MMA directly from tensor memory): saves its shared-memory
  // write and read.  Needs K-major A and free TMEM columns beyond the two
  // partial accumulators (not the 2-CTA 256-column tile, whose partials use
  // all 512 columns).
  constexpr bool ALO = Cfg::kAlo;
  constexpr int kTmemNeed = 2 * Cfg::kMmaN + (ALO ? LO * BK : 0);
  constexpr int kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
  constexpr uint32_t kAloCol = 2 * Cfg::kMmaN;  // first TMEM column of the A_lo stages

  extern __shared__ uint8_t smem_raw_[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_) + 1023) & ~uintptr_t(1023));
  uint8_t* rawA = smem;
  uint8_t* rawB = rawA + RAW * Cfg::kABytes;
  uint8_t* loA = rawB + RAW * Cfg::kBBytes;
  uint8_t* loB = loA + ((SPLIT3 && !ALO) ? LO * Cfg::kABytes : 0);
  float* epi_stage = reinterpret_cast<float*>(smem + Cfg::kRawBytes + Cfg::kLoBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kRawBytes + Cfg::kLoBytes + Cfg::kEpiStageBytes);
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
  if (threadIdx.x == 0) trace_mark(p, 0);

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
  if (warp == 2) ptx::tmem_alloc<CG>(tmem_base_slot, kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  // The TMA producers touch only this CTA's shared memory and barriers, so they
  // start loading before the cluster barrier completes (they wait for it after
  // their loop); every other role needs the peer CTA initialised.
  if constexpr (CG == 2) ptx::cluster_arrive();  // each role waits below
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  if (threadIdx.x == 0) trace_mark(p, 1);

  if (warp < 4) {
    ptx::setmaxnreg_dec<80>();  // producer / MMA / allocator warpgroup
    if (warp != 1) {
      // ---------------------------------------------------------- producers
      // Warps 0, 2, 3 (one lane each) take every third K-iteration: a single
      // issuing thread lands at most about one TMA load per ~0.3 us
      // (scripts/tma_probe.py), which bounds skinny tiles whose stages carry
      // little MMA work; three issuers triple that rate.
      const int pi = warp == 0 ? 0 : warp - 1;
      if (ptx::elect_one()) {
        int s = 0, own = 0;
        uint32_t ph = 0;
        UnitIter ui = units_begin(p, cluster_id, num_clusters);
        Unit u;
        int wi = 0;
        int chunk_ready = -1;  // fused distributed mode: highest B chunk known to be present
        while (units_next(p, num_clusters, ui, u)) {
          if (pi == 0 && p.wave_ctr && u.dp && wi >= 1 && wi < p.full_waves) {
            // Keep the persistent clusters in step at tile boundaries so the
            // concurrently live tiles keep sharing A/B panels in L2.
            atomicAdd(p.wave_ctr, 1u);
            const unsigned target = static_cast<unsigned>(wi) * gridDim.x;
            spin_until(p.wave_ctr, target, false, 256);
          }
          wi += u.dp ? 1 : 0;
          int tmi, tni;
          tile_coords(u.tile, p.tiles_m, p.tiles_n, p.group_m, tmi, tni);
          const int row0 = tmi * Cfg::kTileM + static_cast<int>(rank) * kBMCta;
          const int col0 = tni * Cfg::kTileN + static_cast<int>(rank) * BN_CTA;
          const int rows_here = min(kBMCta, p.m - row0);
          for (int kb = u.kb0; kb < u.kb1; ++kb) {
            if (own == pi) {
              if (p.kflags) {
                const int c = kb / p.kchunk_blocks;
                if (c > chunk_ready) {
                  wait_chunk_flag(p.kflags + c, p.kepoch);
                  chunk_ready = c;
                }
              }
              if (kb == max(u.kb0, u.kb1 - p.kc_blocks) && u.kb0 == 0 && p.beta != 0.0f && rows_here > 0) {
                // This unit ends in the epilogue (a whole tile or a stream-K
                // finalizer) and will read beta*C: stage this CTA's C rows
                // in L2 about one K_c chunk (plus the ring depth) ahead, so the
                // epilogue's loads hit L2 instead of exposing DRAM latency.
                const int c0 = tni * Cfg::kTileN;
                const int cols = min(Cfg::kTileN, p.n - c0);
                const uint32_t bytes = static_cast<uint32_t>(cols * 4) & ~15u;  // floor: never past the row
                if (bytes)
                  for (int r = 0; r < rows_here; ++r) ptx::prefetch_l2_bulk(p.C + (row0 + r) * p.ldc + c0, bytes);
              }
              ptx::mbar_wait(&empty_raw[s], ph ^ 1);
              ptx::mbar_arrive_expect_tx(&full[s], Cfg::kABytes + Cfg::kBBytes);
              if constexpr (CONV) {
                // K-block kb = (filter tap, BK-channel chunk).  Output pixel row0
                // = (b, y, x); its input window starts at (y - pad, x - pad) and
                // the tap adds (ky, kx) as im2col offsets.  TMA walks 128 output
                // pixels in W, H, N order and zero-fills outside the image.
                const int chunks = p.cv_c / BK;
                const int tap = kb / chunks, c0 = (kb - tap * chunks) * BK;
                const int ky = tap / p.cv_s, kx = tap - ky * p.cv_s;
                const int hw = p.cv_ho * p.cv_wo;
                const int b = row0 / hw, yx = row0 - b * hw;
                const int y = yx / p.cv_wo, x = yx - y * p.cv_wo;
                ptx::tma_load_im2col_4d(rawA + s * Cfg::kABytes, &tmA, &full[s], c0, x - p.cv_pad, y - p.cv_pad, b,
                                        static_cast<uint16_t>(kx), static_cast<uint16_t>(ky));
              } else if constexpr (!TA) {  // A: one K-major box BK (k) x 128 (rows)
                ptx::tma_load_2d(rawA + s * Cfg::kABytes, &tmA, &full[s], kb * BK, row0);
              } else if constexpr (BF16) {  // A^T: one un-swizzled box 128 (rows) x 32 (k)
                ptx::tma_load_2d(rawA + s * Cfg::kABytes, &tmA, &full[s], row0, kb * BK);
              } else {              // A^T: four MN-major boxes 32 (rows) x 32 (k)
#pragma unroll
                for (int j = 0; j < kBMCta / 32; ++j)
                  ptx::tma_load_2d(rawA + s * Cfg::kABytes + j * 4096, &tmA, &full[s], row0 + 32 * j, kb * BK);
              }
              if constexpr (!TB && BF16) {  // B: one un-swizzled box BN_CTA (cols) x 32 (k)
                ptx::tma_load_2d(rawB + s * Cfg::kBBytes, &tmB, &full[s], col0, kb * BK);
              } else if constexpr (!TB) {  // B: BN_CTA/32 MN-major boxes 32 (cols) x 32 (k)
#pragma unroll
                for (int j = 0; j < BN_CTA / 32; ++j)
                  ptx::tma_load_2d(rawB + s * Cfg::kBBytes + j * 4096, &tmB, &full[s], col0 + 32 * j, kb * BK);
              } else {              // B^T: one K-major box BK (k) x BN_CTA (cols)
                ptx::tma_load_2d(rawB + s * Cfg::kBBytes, &tmB, &full[s], kb * BK, col0);
              }
            }
            if (++own == kProducers) own = 0;
            if (++s == RAW) { s = 0; ph ^= 1; }
          }
        }
        if (pi == 0) trace_mark(p, 2);  // producer done issuing
      }
      __syncwarp();
      if constexpr (CG == 2) ptx::cluster_wait();  // the barrier phase this warp arrived at on entry
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      if constexpr (CG == 2) ptx::cluster_wait();
      ptx::tc_fence_after();
      if (rank == 0 && ptx::elect_one()) {
        constexpr uint32_t idesc = ptx::idesc_tf32(Cfg::kMmaM, Cfg::kMmaN, /*A MN-major*/ TA ? 1 : 0,
                                                   /*B MN-major*/ TB ? 0 : 1);
        // K-major tile (rows of 128 B = 32 k, SWIZZLE_128B): K step of 8 = 32 B inside the row.
        // MN-major tile (rows of 128 B = 32 m/n, 32-B-atom swizzle): K step of 8 rows = 1024 B
        // (two 512-B atoms, SBO); 32-column atoms 4096 B apart (LBO).
        // BK 16: rows of 64 B (16 k), SWIZZLE_64B, 8-row groups 512 B apart.
        auto desc_k = [](uint32_t base, int ks) {
          return ptx::sdesc(base + ks * 32, 16, 8 * BK * 4, BK == 32 ? ptx::kLayoutSW128 : ptx::kLayoutSW64);
        };
        auto desc_mn = [](uint32_t base, int ks) {
          return ptx::sdesc(base + ks * 1024, 4096, 512, ptx::kLayoutSW128Base32B);
        };
        const uint32_t rawA_s = ptx::smem_u32(rawA), rawB_s = ptx::smem_u32(rawB);
        const uint32_t loA_s = ptx::smem_u32(loA), loB_s = ptx::smem_u32(loB);
        int s = 0, sl = 0, pb = 0;
        uint32_t ph = 0, phl = 0, pph = 0;
        bool first_mma = p.trace != nullptr;
        UnitIter ui = units_begin(p, cluster_id, num_clusters);
        Unit u;
        while (units_next(p, num_clusters, ui, u)) {
          for (int kb0 = u.kb0; kb0 < u.kb1; kb0 += p.kc_blocks) {
            const int kb1 = min(kb0 + p.kc_blocks, u.kb1);
            ptx::mbar_wait_cluster(&part_empty[pb], pph ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + static_cast<uint32_t>(pb * Cfg::kMmaN);
            for (int kb = kb0; kb < kb1; ++kb) {
              ptx::mbar_wait_cluster(&ready[sl], phl);
              ptx::tc_fence_after();
              if (first_mma) { trace_mark(p, 4); first_mma = false; }  // first MMA issue
              if constexpr (BF16) {
                // all nine products a_i * b_j per K = 16 step, smallest first; the
                // three MMAs sharing A plane i read it from shared memory once
                // (collector fill / use / lastuse)
                constexpr uint32_t idesc_b = ptx::idesc_bf16(Cfg::kMmaM, Cfg::kMmaN);
                const uint32_t st0 = loA_s + sl * Cfg::kSplitStage;
#pragma unroll
                for (int ks = 0; ks < BK / 16; ++ks) {
#pragma unroll
                  for (int ia = 2; ia >= 0; --ia) {
                    const uint64_t aD = ptx::sdesc(st0 + ia * Cfg::kPlaneA + ks * 32, 16, 512, ptx::kLayoutSW64);
#pragma unroll
                    for (int ib = 2; ib >= 0; --ib) {
                      const uint64_t bD = ptx::sdesc(st0 + 3 * Cfg::kPlaneA + ib * Cfg::kPlaneB + ks * 32, 16, 512,
                                                     ptx::kLayoutSW64);
                      const uint32_t acc = (kb != kb0 || ks != 0 || ia != 2 || ib != 2) ? 1u : 0u;
                      if (ib == 2) ptx::mma_bf16<CG, 1>(d, aD, bD, idesc_b, acc);
                      else if (ib == 1) ptx::mma_bf16<CG, 3>(d, aD, bD, idesc_b, acc);
                      else ptx::mma_bf16<CG, 2>(d, aD, bD, idesc_b, acc);
                    }
                  }
                }
              } else {
#pragma unroll
              for (int ks = 0; ks < BK / 8; ++ks) {
                const uint64_t aH = TA ? desc_mn(rawA_s + s * Cfg::kABytes, ks) : desc_k(rawA_s + s * Cfg::kABytes, ks);
                const uint64_t bH = TB ? desc_k(rawB_s + s * Cfg::kBBytes, ks) : desc_mn(rawB_s + s * Cfg::kBBytes, ks);
                const uint32_t acc = (kb != kb0 || ks != 0) ? 1u : 0u;  // fresh partial per K_c chunk
                if constexpr (SPLIT3) {
                  const uint64_t aL = TA ? desc_mn(loA_s + sl * Cfg::kABytes, ks) : desc_k(loA_s + sl * Cfg::kABytes, ks);
                  (void)aL;
                  const uint64_t bL = TB ? desc_k(loB_s + sl * Cfg::kBBytes, ks) : desc_mn(loB_s + sl * Cfg::kBBytes, ks);
                  // A_hi feeds two MMAs back to back: fetched from smem once (collector fill/lastuse)
                  if constexpr (ALO) {
                    constexpr uint32_t idesc_k = ptx::idesc_tf32(Cfg::kMmaM, Cfg::kMmaN, 0, TB ? 0 : 1);
                    ptx::mma_tf32_tmem_a<CG>(d, tmem_base + kAloCol + sl * BK + ks * 8, bH, idesc_k, acc);
                  } else {
                    ptx::mma_tf32<CG>(d, aL, bH, idesc, acc);
                  }
                  ptx::mma_tf32<CG, 1>(d, aH, bL, idesc, 1u);
                  ptx::mma_tf32<CG, 2>(d, aH, bH, idesc, 1u);
                } else {
                  ptx::mma_tf32<CG>(d, aH, bH, idesc, acc);
                }
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
        trace_mark(p, 5);  // last MMA issued
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ split
    ptx::setmaxnreg_dec<64>();  // split warpgroup: (80 + 64) * 128 + 184 * 256 = 65536
    if constexpr (CG == 2) ptx::cluster_wait();
    ptx::tc_fence_after();
    const int st = threadIdx.x - 128;
    const uint32_t rawA_s = ptx::smem_u32(rawA), rawB_s = ptx::smem_u32(rawB);
    const uint32_t loA_s = ptx::smem_u32(loA), loB_s = ptx::smem_u32(loB);
    int s = 0, sl = 0;
    uint32_t ph = 0, phl = 0;
    UnitIter ui = units_begin(p, cluster_id, num_clusters);
    Unit u;
    bool first_full = p.trace != nullptr && st == 0;
    while (units_next(p, num_clusters, ui, u)) {
      for (int kb = u.kb0; kb < u.kb1; ++kb) {
        ptx::mbar_wait(&full[s], ph);
        if (first_full) { trace_mark(p, 8); first_full = false; }  // first TMA stage landed
        // The ready ring must not run more than LO stages ahead of the MMA
        // (an mbarrier phase may not complete twice before it is observed).
        ptx::mbar_wait(&empty_lo[sl], phl ^ 1);
        if constexpr (SPLIT3) {
          if constexpr (ALO) {
            // Row r = this thread's TMEM lane (warp w owns lanes 32*(w%4)..+31):
            // read its row of the raw K-major A tile (16-B chunk c of a 128-B
            // row lives at chunk c ^ (r % 8); of a 64-B row at c ^ ((r/2) % 4)),
            // split, store BK columns of A_lo.
            const int r = st;
            const uint32_t rowp = rawA_s + s * Cfg::kABytes + r * (BK * 4);
            uint32_t lo[BK];
#pragma unroll
            for (int c = 0; c < BK / 4; ++c) {
              const int pc = BK == 32 ? (c ^ (r & 7)) : (c ^ ((r >> 1) & 3));
              const uint4 v = ptx::lds128(rowp + (pc << 4));
              lo[4 * c] = tf32_lo_bits(v.x);
              lo[4 * c + 1] = tf32_lo_bits(v.y);
              lo[4 * c + 2] = tf32_lo_bits(v.z);
              lo[4 * c + 3] = tf32_lo_bits(v.w);
            }
            const uint32_t ta = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) + kAloCol + sl * BK;
            if constexpr (BK == 32) ptx::tmem_st_32x32b_x32(ta, lo);
            else ptx::tmem_st_32x32b_x16(ta, lo);
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
          } else {
            split_tile<Cfg::kABytes>(rawA_s + s * Cfg::kABytes, loA_s + sl * Cfg::kABytes, st);
          }
          if constexpr (!TM_MUT(2)) split_tile<Cfg::kBBytes>(rawB_s + s * Cfg::kBBytes, loB_s + sl * Cfg::kBBytes, st);
          else zero_tile<Cfg::kBBytes>(loB_s + sl * Cfg::kBBytes, st);  // mutant: B_lo = 0
          ptx::fence_proxy_async_smem();
        } else if constexpr (BF16) {
          // thread st splits row st of A (128 rows) and, if st < BN_CTA, row st of
          // B^T (B column st) into the three K-major bf16 planes of split slot sl
          const uint32_t dst = loA_s + sl * Cfg::kSplitStage;
          split_row_bf16<!TA>(rawA_s + s * Cfg::kABytes, kBMCta, st, dst, Cfg::kPlaneA);
          if (st < BN_CTA)
            split_row_bf16<TB>(rawB_s + s * Cfg::kBBytes, BN_CTA, st, dst + 3 * Cfg::kPlaneA, Cfg::kPlaneB);
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
    ptx::setmaxnreg_inc<184>();
    if constexpr (CG == 2) ptx::cluster_wait();
    ptx::tc_fence_after();
    const int q = warp & 3;             // TMEM lane quarter (rows 32q..32q+31 of this CTA)
    const int h = (warp - 8) >> 2;      // column half
    int pb = 0;
    uint32_t pph = 0;
    UnitIter ui = units_begin(p, cluster_id, num_clusters);
    Unit u;
    const int wslot = (static_cast<int>(rank) * kEpiWarps + (warp - 8));  // flag slot within a cluster
    while (units_next(p, num_clusters, ui, u)) {
      int tmi, tni;
      tile_coords(u.tile, p.tiles_m, p.tiles_n, p.group_m, tmi, tni);
      float acc[KCOLS];
#pragma unroll
      for (int j = 0; j < KCOLS; ++j) acc[j] = 0.0f;
      for (int kb0 = u.kb0; kb0 < u.kb1; kb0 += p.kc_blocks) {
        ptx::mbar_wait(&part_full[pb], pph);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                               static_cast<uint32_t>(pb * Cfg::kMmaN + h * KCOLS);
        if constexpr (KCOLS >= 16) {
#pragma unroll
          for (int c = 0; c < KCOLS; c += 16) {
            uint32_t r[16];
            ptx::tmem_ld_32x32b_x16(taddr + c, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[c + j] += __uint_as_float(r[j]);  // RN promotion
          }
        } else {
          uint32_t r[8];
          ptx::tmem_ld_32x32b_x8(taddr, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += __uint_as_float(r[j]);  // RN promotion
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) ptx::mbar_arrive_cluster(&part_empty[pb], 0);
          else ptx::mbar_arrive(&part_empty[pb]);
        }
        if (++pb == 2) { pb = 0; pph ^= 1; }
      }
      if (warp == 8 && lane == 0) trace_mark(p, 3);  // last TMEM partial of this unit drained
      // Workspace slice of this warp in a cluster's partial: [rank][warp][KCOLS/4][32 lanes] float4,
      // so every warp-wide access is 512 contiguous bytes; the same warp/lane of
      // every cluster uses the same offsets, so partials line up element by element.
      const long long ws_off = ((static_cast<long long>(rank) * kEpiWarps + (warp - 8)) * (KCOLS / 4)) * 32 + lane;
      const long long ws_stride = static_cast<long long>(CG) * kEpiWarps * (KCOLS / 4) * 32;  // float4 per cluster
      if (u.kb0 > 0) {
        // partial unit: publish the fp32 partial, then the epoch flag
        float4* w = reinterpret_cast<float4*>(p.ws) + cluster_id * ws_stride + ws_off;
#pragma unroll
        for (int j = 0; j < KCOLS / 4; ++j)
          w[j * 32] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(p.flags + cluster_id * (CG * kEpiWarps) + wslot, p.epoch);
        if (warp == 8 && lane == 0) trace_mark(p, 9);  // partial published
        continue;
      }
      if (u.kb1 < p.kblocks) {
        // finalizer: add the partials of the clusters that own the rest of this
        // tile, in increasing cluster order (fixed order -> deterministic)
        const long long tile_end = static_cast<long long>(u.tile + 1) * p.kblocks;
        for (int c2 = cluster_id + 1; c2 < num_clusters && sk_start(p.iters, c2, num_clusters) < tile_end; ++c2) {
          const unsigned* f = p.flags + c2 * (CG * kEpiWarps) + wslot;
          if (lane == 0) {
            spin_until(f, p.epoch, true, 64);
          }
          __syncwarp();
          const unsigned seen = ld_acquire_gpu(f);  // every lane acquires (orders its own loads below)
          (void)seen;
          if (warp == 8 && lane == 0) trace_mark(p, 10);  // (last) partial flag acquired
          const float4* w = reinterpret_cast<const float4*>(p.ws) + c2 * ws_stride + ws_off;
          constexpr int kGrp = (KCOLS / 4) < 8 ? (KCOLS / 4) : 8;
#pragma unroll
          for (int j0 = 0; j0 < KCOLS / 4; j0 += kGrp) {
            float4 v[kGrp];
#pragma unroll
            for (int j = 0; j < kGrp; ++j) v[j] = __ldcg(w + (j0 + j) * 32);
#pragma unroll
            for (int j = 0; j < kGrp; ++j) {
              acc[4 * (j0 + j)] += v[j].x;
              acc[4 * (j0 + j) + 1] += v[j].y;
              acc[4 * (j0 + j) + 2] += v[j].z;
              acc[4 * (j0 + j) + 3] += v[j].w;
            }
          }
        }
      }
      const int wrow0 = tmi * Cfg::kTileM + static_cast<int>(rank) * kBMCta + q * 32;
      const int col0 = tni * Cfg::kTileN + h * KCOLS;
      if (warp == 8 && lane == 0) trace_mark(p, 6);  // accumulation of this unit done
      if (wrow0 < p.m && col0 < p.n)
        epi_store<KCOLS>(p.C, p.ldc, p.m, p.n, wrow0, col0, acc, p.alpha, p.beta,
                         epi_stage + (warp - 8) * 32 * kEpiStride, lane);
      if (warp == 8 && lane == 0) trace_mark(p, 7);  // epilogue of this unit done
    }
  }

  // ---------------------------------------------------------------- teardown
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) ptx::cluster_sync();
  if (threadIdx.x == 0) trace_mark(p, 11);  // teardown barrier passed
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, kTmemCols);
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

// Common launch: p carries the problem (m, n, k, tiles, kblocks, C, alpha,
// beta, and the conv geometry for CONV kernels); this fills the schedule
// (stream-K / wave barrier / tuning knobs) and launches the cluster kernel.
template <int CG, int BN_CTA, int PREC, bool TA, bool TB, int BK, bool CONV>
tm_status launch_kernel(const CUtensorMap& tmA, const CUtensorMap& tmB, TcParams p, int num_sms, bool streamk,
                        cudaStream_t stream) {
  using Cfg = TcCfg<CG, BN_CTA, PREC, BK, TA>;
  auto kern = k_sgemm_tc<CG, BN_CTA, PREC, TA, TB, BK, CONV>;
  static std::atomic<unsigned long long> optin{0};  // per instantiation, bit per device
  if (tm_status st = ensure_smem_optin(optin, kern, Cfg::kSmemBytes); st != TM_OK) return st;
  // Tuning knobs (bench/tests only), read once per process.
  static const int env_kc = [] { const char* e = std::getenv("TM_KC_BLOCKS"); return e ? std::max(1, std::atoi(e)) : 0; }();
  static const int env_gm = [] { const char* e = std::getenv("TM_GROUP_M"); return e ? std::max(1, std::atoi(e)) : 0; }();
  p.kc_blocks = env_kc ? env_kc : kKcBlocksDefault * 32 / BK;  // K_c = 128 elements
  p.group_m = env_gm ? env_gm : kGroupMDefault;
  const int max_clusters = num_sms / CG;
  int clusters = p.num_tiles < max_clusters ? p.num_tiles : max_clusters;
  p.iters = static_cast<long long>(p.num_tiles) * p.kblocks;
  p.streamk = 0;
  p.sk_tiles = 0;
  p.ws = nullptr;
  p.flags = nullptr;
  p.epoch = 0;
  void* graph_owned = nullptr;  // workspace allocated inside a CUDA graph being captured
  if (streamk) {
    clusters = max_clusters;
    // Hybrid: with at least one full wave of tiles, only the partial wave's tiles
    // (mode 1) or the partial wave plus one full wave (mode 2: more stream-K work
    // per cluster) are split; the rest run whole after each cluster's share.
    // Measured (scripts/r02/hybrid_ab.sh, one box): C3 4096^3 0.627 ms pure
    // stream-K -> 0.568 (mode 1) / 0.575 (mode 2); C4 50176x64x576 (18 K-blocks)
    // 39.1 / 39.1 / 37.4 us.  Short-K tiles take mode 2, long-K mode 1;
    // TM_SK_HYBRID=0|1|2 overrides (0: pure stream-K).
    static const int env_hybrid = [] { const char* e = std::getenv("TM_SK_HYBRID"); return e ? std::atoi(e) : -1; }();
    // The region and the cluster count (plan.cpp streamk_region): every cluster
    // owns >= 2 iterations of the region, the remaining tiles form whole waves.
    p.sk_tiles = static_cast<int>(streamk_region(p.num_tiles, p.kblocks, clusters, env_hybrid, &clusters));
    p.iters = static_cast<long long>(p.sk_tiles) * p.kblocks;
    const size_t ws_bytes = static_cast<size_t>(clusters) * CG * kBMCta * Cfg::kMmaN * 4;
    // flags[0] of the workspace is reserved for the wave barrier counter
    const size_t flag_count = 1 + static_cast<size_t>(clusters) * CG * kEpiWarps;
    tm_status st = streamk_workspace(stream, ws_bytes, flag_count, &p.ws, &p.flags, &p.epoch, &graph_owned);
    if (st != TM_OK) return st;
    p.flags += 1;
    p.streamk = 1;
  }

  p.wave_ctr = nullptr;
  p.full_waves = 0;
  // Wave barrier (default on; TM_WAVE_SYNC=0 disables): measured on C5 it cuts
  // DRAM traffic 35 -> 22 GB per launch and, under the power cap, raises the
  // sustained clock and throughput by ~10%.  Only for long K loops: with short
  // tiles (C4, the convolution: <= 18 K-blocks) there is little panel reuse to
  // protect and the per-tile grid-wide barrier costs 10-20%.
  static const bool wave_sync = [] { const char* e = std::getenv("TM_WAVE_SYNC"); return !(e && e[0] == '0'); }();
  const int dp_tiles = p.num_tiles - (p.streamk ? p.sk_tiles : 0);  // hybrid: whole waves only
  if (wave_sync && !CONV && p.kblocks >= 64 && dp_tiles / clusters >= 2) {
    if (p.streamk) {
      p.wave_ctr = p.flags - 1;  // slot 0 of the stream-K flags (reserved above)
    } else {
      float* ws_unused = nullptr;
      unsigned epoch_unused = 0;
      tm_status st = streamk_workspace(stream, 0, 1, &ws_unused, &p.wave_ctr, &epoch_unused, &graph_owned);  // slot 0
      if (st != TM_OK) return st;
    }
    if (cudaMemsetAsync(p.wave_ctr, 0, sizeof(unsigned), stream) != cudaSuccess) return TM_ERR_CUDA;
    p.full_waves = dp_tiles / clusters;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * CG, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // Stream-K finalizers and the wave barrier wait on other CTAs: require the
  // whole (persistent, <= one CTA per SM) grid to be co-resident.  Nsight
  // Compute cannot replay cooperative cluster launches; TM_COOPERATIVE=0 drops
  // only this launch-time check for profiling runs (same kernel, same barrier).
  static const bool coop = [] { const char* e = std::getenv("TM_COOPERATIVE"); return !(e && e[0] == '0'); }();
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = (coop && (p.streamk || p.wave_ctr)) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  p.trace = nullptr;
  const char* trace_path = std::getenv("TM_TRACE_PATH");  // debug timeline (bench/profiling only)
  if (trace_path) {
    if (cudaMalloc(&p.trace, sizeof(unsigned long long) * kTraceSlots * clusters * CG) != cudaSuccess) return TM_ERR_CUDA;
    cudaMemsetAsync(p.trace, 0, sizeof(unsigned long long) * kTraceSlots * clusters * CG, stream);
  }
  const bool launched = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, p) == cudaSuccess;
  if (graph_owned && cudaFreeAsync(graph_owned, stream) != cudaSuccess) return TM_ERR_CUDA;
  if (!launched) return TM_ERR_CUDA;
  if (trace_path) {
    const int n = kTraceSlots * clusters * CG;
    unsigned long long* h = new unsigned long long[n];
    cudaStreamSynchronize(stream);
    cudaMemcpy(h, p.trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
    cudaFree(p.trace);
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "{\"cg\":%d,\"bn\":%d,\"sk\":%d,\"m\":%d,\"n\":%d,\"k\":%d,\"ctas\":%d,\"t\":[", CG, BN_CTA,
                   p.streamk, p.m, p.n, p.k, clusters * CG);
      for (int i = 0; i < n; ++i) std::fprintf(f, "%s%llu", i ? "," : "", h[i]);
      std::fprintf(f, "]}\n");
      std::fclose(f);
    }
    delete[] h;
  }
  return TM_OK;
}

template <int CG, int BN_CTA, int PREC, bool TA, bool TB>
tm_status launch_cfg(const GemmArgs& a, int num_sms, bool streamk, cudaStream_t stream) {
  using Cfg = TcCfg<CG, BN_CTA, PREC>;
  CUtensorMap tmA, tmB;
  // K-major operands (A, B^T): box 32 (k) x rows, SWIZZLE_128B.  MN-major
  // operands (A^T, B): box 32 (m or n) x 32 (k), 128-B swizzle with 32-B atoms
  // for the tf32 MMAs; BF16x9 reads MN-major raw tiles only in its split
  // warps, so it loads them as one un-swizzled box (128 or BN_CTA) x 32 (k).
  constexpr bool BF16 = PREC == kPrecBf16x9;
  bool ok;
  if constexpr (!TA) ok = encode_2d(&tmA, a.A, a.m, a.k, a.lda, kBK, kBMCta, CU_TENSOR_MAP_SWIZZLE_128B);
  else if constexpr (BF16) ok = encode_2d(&tmA, a.A, a.k, a.m, a.lda, kBMCta, kBK, CU_TENSOR_MAP_SWIZZLE_NONE);
  else ok = encode_2d(&tmA, a.A, a.k, a.m, a.lda, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!ok) return TM_ERR_INTERNAL;
  if constexpr (!TB && BF16) ok = encode_2d(&tmB, a.B, a.k, a.n, a.ldb, BN_CTA, kBK, CU_TENSOR_MAP_SWIZZLE_NONE);
  else if constexpr (!TB) ok = encode_2d(&tmB, a.B, a.k, a.n, a.ldb, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  else ok = encode_2d(&tmB, a.B, a.n, a.k, a.ldb, kBK, BN_CTA, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!ok) return TM_ERR_INTERNAL;
  TcParams p{};
  p.A = a.A;
  p.lda = a.lda;
  p.m = static_cast<int>(a.m);
  p.n = static_cast<int>(a.n);
  p.k = static_cast<int>(a.k);
  p.tiles_m = static_cast<int>((a.m + Cfg::kTileM - 1) / Cfg::kTileM);
  p.tiles_n = static_cast<int>((a.n + Cfg::kTileN - 1) / Cfg::kTileN);
  p.num_tiles = p.tiles_m * p.tiles_n;
  p.kblocks = static_cast<int>((a.k + kBK - 1) / kBK);
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.C = a.C;
  p.ldc = a.ldc;
  p.kflags = a.kflags;
  p.kepoch = a.kepoch;
  p.kchunk_blocks = static_cast<int>(a.kchunk / kBK);
  if (a.kflags && (a.kchunk <= 0 || a.kchunk % kBK != 0)) return TM_ERR_INVALID_VALUE;
  return launch_kernel<CG, BN_CTA, PREC, TA, TB, 32, false>(tmA, tmB, p, num_sms, streamk, stream);
}

template <int PREC, bool TA, bool TB>
tm_status launch_split(const GemmArgs& a, int cg, int bn, int num_sms, bool sk, cudaStream_t s) {
  if constexpr (PREC == kPrecBf16x9) {
    // BF16x9 is compiled for 64- and 128-column CTA tiles (32 -> 64)
    if (bn == 32) bn = 64;
    if (cg == 2 && bn == 128) return launch_cfg<2, 128, PREC, TA, TB>(a, num_sms, sk, s);
    if (cg == 2 && bn == 64) return launch_cfg<2, 64, PREC, TA, TB>(a, num_sms, sk, s);
    if (cg == 1 && bn == 128) return launch_cfg<1, 128, PREC, TA, TB>(a, num_sms, sk, s);
    if (cg == 1 && bn == 64) return launch_cfg<1, 64, PREC, TA, TB>(a, num_sms, sk, s);
    return TM_ERR_INVALID_VALUE;
  } else {
    if (cg == 2) {
      if (bn == 128) return launch_cfg<2, 128, PREC, TA, TB>(a, num_sms, sk, s);
      if (bn == 64) return launch_cfg<2, 64, PREC, TA, TB>(a, num_sms, sk, s);
      if (bn == 32) return launch_cfg<2, 32, PREC, TA, TB>(a, num_sms, sk, s);
    } else if (cg == 1) {
      if (bn == 128) return launch_cfg<1, 128, PREC, TA, TB>(a, num_sms, sk, s);
      if (bn == 64) return launch_cfg<1, 64, PREC, TA, TB>(a, num_sms, sk, s);
      if (bn == 32) return launch_cfg<1, 32, PREC, TA, TB>(a, num_sms, sk, s);
    }
    return TM_ERR_INVALID_VALUE;
  }
}

}  // namespace

// Tensor-core launch for one operand layout (explicitly instantiated in
// tc_gemm_{nn,nt,tn,tt}.cu): 3xTF32, the single-pass 1xTF32 precision variant
// (one MMA per K step on the raw operands) or BF16x9.
template <bool TA, bool TB>
tm_status launch_tc_op(const GemmArgs& a, const TcChoice& c, int num_sms, cudaStream_t stream) {
  if (a.m > INT32_MAX / 2 || a.n > INT32_MAX / 2 || a.k > INT32_MAX / 2) return TM_ERR_INVALID_VALUE;
  switch (c.prec) {
    case kPrecTf32x3: return launch_split<kPrecTf32x3, TA, TB>(a, c.cg, c.bn_cta, num_sms, c.streamk, stream);
    case kPrecTf32x1: return launch_split<kPrecTf32x1, TA, TB>(a, c.cg, c.bn_cta, num_sms, c.streamk, stream);
    case kPrecBf16x9: return launch_split<kPrecBf16x9, TA, TB>(a, c.cg, c.bn_cta, num_sms, c.streamk, stream);
    default: return TM_ERR_INVALID_VALUE;
  }
}

}  // namespace tmk
