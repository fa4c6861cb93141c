// tc_conv_direct.cu -- direct (halo-tile) 3xTF32 tensor-core convolution for
// few channels and filters (the Conv
// benchmark: 32 x 512 x 512 x 16 input, 16 filters of 3 x 3 x 16).
//
// Same arithmetic as the implicit-GEMM path (tc_conv.cu): M = output pixels,
// N = filters, K = (ky, kx, c) in KRSC order; products of the 3xTF32 split
// accumulated in TMEM over K_c = 128 and promoted with RN adds in registers.
// What differs is how A reaches the tensor core.  The im2col path lands one
// TMA box per (tap, 16 channels) -- 9 boxes of 128 x 64 B per tile for the
// paper's shape -- and is bound by the TMA issue rate (scripts/tma_probe.py).
// Here one 4-D tiled TMA box per tile brings the input "halo" -- R input rows x
// (128 + S - 1) pixels x up to 32 channels, borders zero-filled by the TMA --
// and the split warps build each tap's A operand from it: thread r (TMEM lane
// r = output pixel x0 + r) reads pixel r + kx of halo row ky, splits it into
// hi / lo and stores both into a TMEM stage, from which the MMAs read A.  The
// filters (all of K x BN) stay resident in shared memory, hi and lo, for the
// whole persistent CTA.
//
// Warp roles (512 threads, one CTA per SM, persistent over tiles):
//   warps 0, 2, 3  halo producers (one lane each, tiles round-robin); warp 0
//                  also loads the resident filters once.  Warp 2 allocates TMEM.
//   warp 1         MMA issuer: per (tap, 16 channels) stage, K steps of 8, the
//                  three products A_lo B_hi + A_hi B_lo + A_hi B_hi.
//   warps 4-11     split, two warpgroups taking alternate pairs of stages:
//                  halo -> (hi | lo) TMEM stages (up to 12-deep ring).  One
//                  group alone is latency-bound (~28% issue utilisation).
//   warps 12-15    promotion + epilogue (tc_gemm.cuh epi_store: alpha / beta,
//                  full / partial tile separation), all BN columns per warp.
#include "tc_gemm.cuh"

namespace tmk {
namespace {

constexpr int kDcBK = 16;        // channels per stage (16 = one 64-B filter box row)
constexpr int kDcPix = 128;      // output pixels per tile = TMEM lanes
constexpr int kDcPb = 4;         // TMEM partial accumulators (BN columns each)
constexpr int kDcSplitWarps = 8; // two split warpgroups
constexpr int kDcEpiWarps = 4;   // one promotion/epilogue warpgroup (all BN columns per warp)
constexpr int kDcMaxSmem = 227 * 1024;

struct DcParams {
  int nb, h, w, c, f, r, s, pad, ho, wo;
  int tiles_x, num_tiles, kblocks, kc_blocks, chunks;  // chunks = c / 16
  int cw;              // channels per halo box (16 or 32)
  int halo_w;          // 128 + s - 1 pixels
  int box_bytes;       // one halo box (r x halo_w x cw floats) rounded up to 1 KiB
  int slot_bytes;      // (c / cw) boxes
  int n_slots;         // halo ring depth
  int bres_bytes;      // resident filters, hi (same again for lo)
  float alpha, beta;
  float* Y;
  unsigned long long* trace;  // debug timeline of CTA 0 [kDcTraceTiles][kDcTraceEv] (%globaltimer) or null
};

constexpr int kDcTraceTiles = 32, kDcTraceEv = 8;
// events: 0 halo issued, 1 split saw halo, 2 MMA saw first ready, 3 MMA last commit issued,
//         4 epilogue saw last partial, 5 epilogue stored, 6 split last ready arrive, 7 MMA saw last ready
// Compiled in only with -DTM_DC_TRACE (the marks sit in the per-stage loops).
#ifdef TM_DC_TRACE
#define DC_MARK(p, t, ev) dc_mark(p, ((t) - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x), ev)
#else
#define DC_MARK(p, t, ev) ((void)0)
#endif
__device__ __forceinline__ void dc_mark(const DcParams& p, int i, int ev) {
  if (p.trace && blockIdx.x == 0 && i < kDcTraceTiles) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[i * kDcTraceEv + ev] = t;
  }
}

template <int BN>
struct DcCfg {
  static constexpr int kBBox = BN * kDcBK * 4;  // one K-block of filters: BN rows x 64 B (SWIZZLE_64B)
  static constexpr int kCols = BN;              // output columns per promotion warp
  static constexpr int kAcol = kDcPb * BN;      // first TMEM column of the A stages
  static constexpr int kSlotCols = 2 * 2 * kDcBK;  // ring slot: two stages of (16 hi | 16 lo) columns
  static constexpr int kLo0 = (512 - kAcol) / kSlotCols;
  static constexpr int kLo = kLo0 < 6 ? kLo0 : 6;  // TMEM A ring slots
  static constexpr int kTmemNeed = kAcol + kLo * kSlotCols;
  static constexpr int kTmemCols = kTmemNeed <= 256 ? 256 : 512;
  static constexpr int kEpiBytes = kEpiWarps * 32 * kEpiStride * 4;
};

// Wait for a phase with a back-off: for roles that wait long (producers for a
// free halo slot, the epilogue for a finished accumulator), so that their
// polling does not take issue slots from the split warps on the same SM
// sub-partition.
__device__ __forceinline__ void dc_wait_lazy(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  while (!ptx::mbar_try_wait(a, parity)) __nanosleep(128);
}

__device__ __forceinline__ void dc_tile(const DcParams& p, int t, int& b, int& y, int& x0) {
  const int xt = t % p.tiles_x;
  const int rest = t / p.tiles_x;
  y = rest % p.ho;
  b = rest / p.ho;
  x0 = xt * kDcPix;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_direct(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, DcParams p) {
  using Cfg = DcCfg<BN>;
  constexpr int KCOLS = Cfg::kCols;
  extern __shared__ uint8_t smem_raw_[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_) + 1023) & ~uintptr_t(1023));
  uint8_t* bres = smem;
  uint8_t* bres_lo = bres + p.bres_bytes;
  uint8_t* halo = bres_lo + p.bres_bytes;
  float* epi_stage = reinterpret_cast<float*>(halo + p.n_slots * p.slot_bytes);
  uint64_t* bres_full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi_stage) + Cfg::kEpiBytes);
  uint64_t* halo_full = bres_full + 1;         // [n_slots] TMA landed
  uint64_t* halo_empty = halo_full + p.n_slots;  // [n_slots] split warps done reading
  uint64_t* ready = halo_empty + p.n_slots;    // [Cfg::kLo] TMEM A stage written
  uint64_t* empty_lo = ready + Cfg::kLo;          // [Cfg::kLo] MMAs done with the stage (commit)
  uint64_t* part_full = empty_lo + Cfg::kLo;  // [kDcPb] TMEM partial complete (commit)
  uint64_t* part_empty = part_full + kDcPb;   // [kDcPb] partial drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(part_empty + kDcPb);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bres_full, 1);
    for (int i = 0; i < p.n_slots; ++i) {
      ptx::mbar_init(&halo_full[i], 1);
      ptx::mbar_init(&halo_empty[i], kDcSplitWarps);
    }
    for (int i = 0; i < Cfg::kLo; ++i) {
      ptx::mbar_init(&ready[i], kSplitThreads / 32);
      ptx::mbar_init(&empty_lo[i], 1);
    }
    for (int i = 0; i < kDcPb; ++i) {
      ptx::mbar_init(&part_full[i], 1);
      ptx::mbar_init(&part_empty[i], kDcEpiWarps);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmW);
  }
  if (warp == 2) ptx::tmem_alloc<1>(tmem_slot, Cfg::kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    ptx::setmaxnreg_dec<80>();
    if (warp != 1) {
      // ------------------------------------------------------------ producers
      const int pi = warp == 0 ? 0 : warp - 1;
      if (ptx::elect_one()) {
        if (pi == 0) {
          ptx::mbar_arrive_expect_tx(bres_full, static_cast<uint32_t>(p.kblocks * Cfg::kBBox));
          for (int kb = 0; kb < p.kblocks; ++kb)
            ptx::tma_load_2d(bres + kb * Cfg::kBBox, &tmW, bres_full, kb * kDcBK, 0);
        }
        int slot = 0, own = 0;
        uint32_t ph = 0;
        const int boxes = p.c / p.cw;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
          if (own == pi) {
            int b, y, x0;
            dc_tile(p, t, b, y, x0);
            ptx::mbar_wait(&halo_empty[slot], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&halo_full[slot], static_cast<uint32_t>(boxes * p.r * p.halo_w * p.cw * 4));
            for (int i = 0; i < boxes; ++i)
              ptx::tma_load_4d(halo + slot * p.slot_bytes + i * p.box_bytes, &tmX, &halo_full[slot], i * p.cw,
                               x0 - p.pad, y - p.pad, b);
            DC_MARK(p, t, 0);
          }
          if (++own == kProducers) own = 0;
          if (++slot == p.n_slots) { slot = 0; ph ^= 1; }
        }
      }
    } else if (ptx::elect_one()) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = ptx::idesc_tf32(kDcPix, BN, 0, 0);
      const uint32_t bres_s = ptx::smem_u32(bres), blo_s = ptx::smem_u32(bres_lo);
      int sl = 0, pb = 0;
      uint32_t phl = 0, pph = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        for (int kb0 = 0; kb0 < p.kblocks; kb0 += p.kc_blocks) {
          const int kb1 = min(kb0 + p.kc_blocks, p.kblocks);
          ptx::mbar_wait(&part_empty[pb], pph ^ 1);
          ptx::tc_fence_after();
          const uint32_t d = tmem_base + static_cast<uint32_t>(pb * BN);
          for (int kb = kb0; kb < kb1; kb += 2) {  // one ring slot = the split's pair of stages
            const int nst = min(2, p.kblocks - kb);
            ptx::mbar_wait(&ready[sl], phl);
            ptx::tc_fence_after();
            if (kb == 0) DC_MARK(p, t, 2);
            if (kb + nst == p.kblocks) DC_MARK(p, t, 7);
            for (int u = 0; u < nst; ++u) {
              const uint32_t a_hi = tmem_base + Cfg::kAcol + sl * Cfg::kSlotCols + u * 2 * kDcBK;
              const uint32_t a_lo = a_hi + kDcBK;
              const int k = kb + u;
#pragma unroll
              for (int ks = 0; ks < kDcBK / 8; ++ks) {
                const uint64_t bH = ptx::sdesc(bres_s + k * Cfg::kBBox + ks * 32, 16, 512, ptx::kLayoutSW64);
                const uint64_t bL = ptx::sdesc(blo_s + k * Cfg::kBBox + ks * 32, 16, 512, ptx::kLayoutSW64);
                const uint32_t acc = (k != kb0 || ks != 0) ? 1u : 0u;
                ptx::mma_tf32_tmem_a<1>(d, a_lo + ks * 8, bH, idesc, acc);
                ptx::mma_tf32_tmem_a<1>(d, a_hi + ks * 8, bL, idesc, 1u);
                ptx::mma_tf32_tmem_a<1>(d, a_hi + ks * 8, bH, idesc, 1u);
              }
            }
            ptx::mma_commit<1>(&empty_lo[sl]);
            if (++sl == Cfg::kLo) { sl = 0; phl ^= 1; }
          }
          ptx::mma_commit<1>(&part_full[pb]);
          if (++pb == kDcPb) { pb = 0; pph ^= 1; }
        }
        DC_MARK(p, t, 3);
      }
    }
  } else if (warp < 12) {
    // -------------------------------------------------------------- split
    // Two split warpgroups (warps 4-7, 8-11) take alternate stage pairs; both
    // keep the launch's 128 registers: (80 + 2 * 128) * 128 + 176 * 128 = 65536.
    const int g = (warp - 4) >> 2;
    const int st = (warp & 3) * 32 + lane;  // = TMEM lane = output pixel x0 + st of the tile
    if (g == 0) {
      // resident filters: lo = split of hi, in place layout (elementwise)
      ptx::mbar_wait(bres_full, 0);
      const uint32_t src = ptx::smem_u32(bres), dst = ptx::smem_u32(bres_lo);
      for (int i = st; i < p.bres_bytes / 16; i += kSplitThreads) ptx::sts128(dst + i * 16, tf32_lo4(ptx::lds128(src + i * 16)));
      ptx::fence_proxy_async_smem();
    }
    const uint32_t halo_s = ptx::smem_u32(halo);
    const uint32_t trow = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) + Cfg::kAcol;
    const bool cw16 = p.cw == 16;          // 64-B halo rows (SWIZZLE_64B), else 128-B rows (SWIZZLE_128B)
    const int rb = p.cw * 4;
    int slot = 0, sl = 0, pair = 0;
    uint32_t ph = 0, phl = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      ptx::mbar_wait(&halo_full[slot], ph);
      if (g == 0 && st == 0) DC_MARK(p, t, 1);
      const uint32_t hb = halo_s + slot * p.slot_bytes;
      int ky = 0, kx = 0, ci = 0;  // K-block kb = (ky * S + kx) * chunks + ci (KRSC order)
      // Two stages per round: both stages' shared loads in flight together,
      // one tcgen05.wait::st for the pair.  Rounds alternate between the groups.
      for (int kb = 0; kb < p.kblocks; kb += 2, ++pair) {
        const int nst = min(2, p.kblocks - kb);
        if ((pair & 1) != g) {  // the other group's round: advance the cursors only
          for (int u = 0; u < nst; ++u) {
            if (++ci == p.chunks) {
              ci = 0;
              if (++kx == p.s) { kx = 0; ++ky; }
            }
          }
          if (++sl == Cfg::kLo) { sl = 0; phl ^= 1; }
          continue;
        }
        uint4 v[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u < nst) {
            const int box = cw16 ? ci : (ci >> 1);
            const int within = cw16 ? 0 : ((ci & 1) << 2);      // first 16-B chunk of these 16 channels
            const int row = ky * p.halo_w + st + kx;             // pixel row inside the box
            const uint32_t rowp = hb + box * p.box_bytes + row * rb;
            // TMA swizzle (box bases 1 KiB aligned): 16-B chunk j of a row is
            // stored at j ^ ((row / 2) % 4) for 64-B rows, j ^ (row % 8) for 128-B rows.
            const int sw = cw16 ? ((row >> 1) & 3) : (row & 7);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[u][j] = ptx::lds128(rowp + (((within + j) ^ sw) << 4));
            if (++ci == p.chunks) {
              ci = 0;
              if (++kx == p.s) { kx = 0; ++ky; }
            }
          }
        }
        ptx::mbar_wait(&empty_lo[sl], phl ^ 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u < nst) {
            uint32_t hl[32];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t x[4] = {v[u][j].x, v[u][j].y, v[u][j].z, v[u][j].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                hl[4 * j + e] = x[e] & 0xFFFFE000u;
                hl[kDcBK + 4 * j + e] = tf32_lo_bits(x[e]);
              }
            }
            ptx::tmem_st_32x32b_x32(trow + sl * Cfg::kSlotCols + u * 2 * kDcBK, hl);
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ready[sl]);
        if (st == 0 && kb + nst == p.kblocks) DC_MARK(p, t, 6);
        if (++sl == Cfg::kLo) { sl = 0; phl ^= 1; }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&halo_empty[slot]);
      if (++slot == p.n_slots) { slot = 0; ph ^= 1; }
    }
  } else {
    // -------------------------------------------------------------- promotion + epilogue
    ptx::setmaxnreg_inc<176>();
    const int q = warp & 3;
    constexpr int h = 0;
    int pb = 0;
    uint32_t pph = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      float acc[KCOLS];
#pragma unroll
      for (int j = 0; j < KCOLS; ++j) acc[j] = 0.0f;
      for (int kb0 = 0; kb0 < p.kblocks; kb0 += p.kc_blocks) {
        ptx::mbar_wait(&part_full[pb], pph);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(pb * BN + h * KCOLS);
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
        if (lane == 0) ptx::mbar_arrive(&part_empty[pb]);
        if (++pb == kDcPb) { pb = 0; pph ^= 1; }
      }
      if (warp == 12 && lane == 0) DC_MARK(p, t, 4);
      int b, y, x0;
      dc_tile(p, t, b, y, x0);
      const int pix0 = (b * p.ho + y) * p.wo + x0;            // first output pixel (GEMM row) of the tile
      const int valid = min(kDcPix, p.wo - x0);               // pixels of this output row in the tile
      const int col0 = h * KCOLS;
      if (q * 32 < valid && col0 < p.f)
        epi_store<KCOLS>(p.Y, p.f, pix0 + valid, p.f, pix0 + q * 32, col0, acc, p.alpha, p.beta,
                         epi_stage + (warp - 12) * 32 * kEpiStride, lane);
      if (warp == 12 && lane == 0) DC_MARK(p, t, 5);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem_base, Cfg::kTmemCols);
  }
}

// NHWC input {C, W, H, N}, box {cw, halo_w, r, 1}: one tile's input rows.
bool encode_halo(CUtensorMap* map, const ConvArgs& a, int cw, int halo_w, int rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(a.c), static_cast<cuuint64_t>(a.w), static_cast<cuuint64_t>(a.h),
                        static_cast<cuuint64_t>(a.nb)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(a.c) * 4, static_cast<cuuint64_t>(a.c * a.w) * 4,
                           static_cast<cuuint64_t>(a.c * a.w * a.h) * 4};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(cw), static_cast<cuuint32_t>(halo_w), static_cast<cuuint32_t>(rows), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(a.X), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, cw == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int dc_bn(int64_t f) { return f <= 16 ? 16 : f <= 32 ? 32 : 64; }

// Fills p and returns the dynamic shared-memory size, or 0 if the shape does
// not fit the direct kernel.
int dc_plan(const ConvArgs& a, DcParams& p) {
  if (a.c % kDcBK != 0 || a.f > 64 || a.r > 32 || a.s > 32) return 0;
  const int64_t ho = a.ho(), wo = a.wo();
  if (ho <= 0 || wo <= 0) return 0;
  const int bn = dc_bn(a.f);
  p = DcParams{};
  p.nb = static_cast<int>(a.nb);
  p.h = static_cast<int>(a.h);
  p.w = static_cast<int>(a.w);
  p.c = static_cast<int>(a.c);
  p.f = static_cast<int>(a.f);
  p.r = static_cast<int>(a.r);
  p.s = static_cast<int>(a.s);
  p.pad = static_cast<int>(a.pad);
  p.ho = static_cast<int>(ho);
  p.wo = static_cast<int>(wo);
  p.tiles_x = static_cast<int>((wo + kDcPix - 1) / kDcPix);
  const int64_t tiles = a.nb * ho * p.tiles_x;
  if (tiles > INT32_MAX / 2 || a.nb * ho * wo > INT32_MAX / 2) return 0;
  p.num_tiles = static_cast<int>(tiles);
  p.chunks = p.c / kDcBK;
  p.kblocks = p.r * p.s * p.chunks;
  p.kc_blocks = kKcBlocksDefault * 32 / kDcBK;  // K_c = 128 (even: chunks end on stage pairs)
  p.cw = p.c % 32 == 0 ? 32 : 16;
  p.halo_w = kDcPix + p.s - 1;
  p.box_bytes = (p.r * p.halo_w * p.cw * 4 + 1023) / 1024 * 1024;
  p.slot_bytes = (p.c / p.cw) * p.box_bytes;
  p.bres_bytes = p.kblocks * bn * kDcBK * 4;
  const int fixed = 1024 + 2 * p.bres_bytes + kEpiWarps * 32 * kEpiStride * 4 + 512;
  const int slots = (kDcMaxSmem - fixed) / p.slot_bytes;
  if (slots < 2) return 0;
  p.n_slots = slots < 4 ? slots : 4;
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.Y = a.Y;
  return fixed + p.n_slots * p.slot_bytes;
}

template <int BN>
tm_status launch_dc(const ConvArgs& a, const DcParams& p, int smem, int num_sms, cudaStream_t stream) {
  CUtensorMap tmX, tmW;
  if (!encode_halo(&tmX, a, p.cw, p.halo_w, static_cast<int>(a.r))) return TM_ERR_INTERNAL;
  const int64_t K = a.r * a.s * a.c;
  if (!encode_2d(&tmW, a.Wt, a.f, K, K, kDcBK, BN, CU_TENSOR_MAP_SWIZZLE_64B)) return TM_ERR_INTERNAL;
  auto kern = k_conv_direct<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kDcMaxSmem) != cudaSuccess)
      return TM_ERR_CUDA;
    attr_set = true;
  }
  const int grid = p.num_tiles < num_sms ? p.num_tiles : num_sms;
  DcParams pp = p;
  const char* trace_path = std::getenv("TM_TRACE_PATH");  // debug timeline (profiling only)
  const int nt = kDcTraceTiles * kDcTraceEv;
  if (trace_path) {
    if (cudaMalloc(&pp.trace, sizeof(unsigned long long) * nt) != cudaSuccess) return TM_ERR_CUDA;
    cudaMemsetAsync(pp.trace, 0, sizeof(unsigned long long) * nt, stream);
  }
  kern<<<grid, kThreads, smem, stream>>>(tmX, tmW, pp);
  if (cudaPeekAtLastError() != cudaSuccess) return TM_ERR_CUDA;
  if (trace_path) {
    unsigned long long h[kDcTraceTiles * kDcTraceEv];
    cudaStreamSynchronize(stream);
    cudaMemcpy(h, pp.trace, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(pp.trace);
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "{\"kernel\":\"conv_direct\",\"bn\":%d,\"ev\":%d,\"t\":[", BN, kDcTraceEv);
      for (int i = 0; i < nt; ++i) std::fprintf(f, "%s%llu", i ? "," : "", h[i]);
      std::fprintf(f, "]}\n");
      std::fclose(f);
    }
  }
  return TM_OK;
}

}  // namespace

bool conv_direct_fits(const ConvArgs& a) {
  DcParams p;
  return dc_plan(a, p) > 0;
}

tm_status launch_conv_direct(const ConvArgs& a, int num_sms, cudaStream_t stream) {
  DcParams p;
  const int smem = dc_plan(a, p);
  if (smem == 0) return TM_ERR_INVALID_VALUE;
  switch (dc_bn(a.f)) {
    case 16: return launch_dc<16>(a, p, smem, num_sms, stream);
    case 32: return launch_dc<32>(a, p, smem, num_sms, stream);
    default: return launch_dc<64>(a, p, smem, num_sms, stream);
  }
}

}  // namespace tmk
