// tc_conv_direct.cu -- direct (halo-tile, shifted-accumulate) 3xTF32
// tensor-core convolution for few channels and filters (SURVEY.md 8(f) item
// 2, the Conv benchmark: 32 x 512 x 512 x 16 input, 16
// filters of 3 x 3 x 16).
//
// Same products as the implicit-GEMM path (tc_conv.cu) -- the 3xTF32 split
// A_lo B_hi + A_hi B_lo + A_hi B_hi, accumulated in TMEM, promoted with RN
// adds in registers -- but a different factorisation of the sum over
// (ky, kx, c).  Output pixel x of filter f is
//     Y[x, f] = sum_kx Z[x + kx, (f, kx)],  Z[p, (f, kx)] = sum_{ky, c} X[p, ky, c] W[f, ky, kx, c],
// where p runs over the tile's input "halo" pixels.  Z is one GEMM with
// M = 128 halo pixels (TMEM lanes), N = F_pad * S columns (filter, tap kx)
// and K = R * C (ky, c); the A operand is the halo itself, with no shifted
// copies, and the kx shift is applied afterwards in registers: lane p adds
// the (f, kx) column of lane p + kx (warp shuffles).  Against the per-tap
// formulation (R * S stages of 16 channels per tile) the split handles S
// times less data and the pipeline S times fewer stages.  Warp q's 32 lanes
// cover halo pixels OW*q .. OW*q + 31 and produce OW = 33 - S outputs, so the
// shift never crosses a warp.
//
// The K = R * C reduction runs in PASSES of RPP filter rows (all R rows in one
// pass when TMEM and shared memory allow; 9x9 takes three passes of 3 rows):
// one 4-D tiled TMA box per (tile, pass) brings the halo rows of the pass --
// RPP input rows x (3 OW + 32) pixels x up to 32 channels, image borders
// zero-filled by the TMA -- and the split writes them into one TMEM A slot;
// the MMA chain of a tile spans its passes' slots.  The filters, rearranged by
// the TMA box itself into B^T rows (kx, f) x 16 channels per (ky, 16-channel)
// stage, stay resident in shared memory, hi and lo, for the whole persistent
// CTA.  Accumulator column kx * F_pad + f holds Z[., (f, kx)], so the shift-add
// reads 16 filters of one kx per TMEM load, whatever S.
//
// Warp roles (512 threads, one CTA per SM, persistent over tiles):
//   warps 0, 2     halo producers (one lane each, alternate tiles); warp 0
//                  also loads the filters once.  Warp 2 allocates TMEM.
//   warp 1         MMA issuer (one lane).
//   warps 4-7      split: halo -> (hi | lo) TMEM A slots, one slot per (tile, pass).
//   warps 8-15     promotion, shift-add and epilogue, two warpgroups, one per
//                  TMEM accumulator (tc_gemm.cuh epi_store: alpha / beta,
//                  full / partial tile separation).  The epilogue is the
//                  longest per-tile chain, hence two groups.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "tc_gemm.cuh"

namespace tmk {
namespace {

constexpr int kDcBK = 16;            // channels per stage (one 64-B row of a filter box)
constexpr int kDcLanes = 128;        // halo pixels per tile = TMEM lanes
constexpr int kDcSplitWarps = 4;     // one split warpgroup
constexpr int kDcEpiWarps = 8;       // two promotion / epilogue warpgroups (one per accumulator)
constexpr int kDcMaxSlots = 4;       // TMEM A slots (one tile each)
constexpr int kDcMaxStages = 8;      // stages (16-channel rows) per pass: RPP * C / 16
constexpr int kDcMaxSmem = 227 * 1024;
// The halo producers alternate tiles by parity and the halo ring depth is
// even, so every ring slot is always filled by the same producer: each slot's
// phases then complete in order, which the parity waits rely on.
constexpr int kDcProducers = 2;

struct DcParams {
  int nb, h, w, c, f, r, pad, ho, wo;
  int fp;              // filters padded to a multiple of 16
  int n;               // MMA N = fp * S (S: the taps of this launch)
  int ow;              // outputs per warp = 33 - (full filter width)
  int kx0;             // first filter column kx of this launch (kx split: 0, then S of the first)
  int tiles_x, num_tiles;
  int chunks;          // c / 16
  int stages;          // rin * chunks: K = 16 * stages (resident filter stages)
  int ro;              // output rows per tile (1, or 2 when the MMA N of one row is small)
  int rin;             // input rows per tile: r + ro - 1
  int ho_t;            // tile rows per image: ceil(ho / ro)
  int nrow;            // MMA N of one output row: fp * S
  int fstages;         // raw filter boxes r * chunks (ro == 2: staged, then expanded)
  int fbox;            // one raw filter box: nrow rows x 64 B
  int fgap;            // bytes between the halo ring and the barriers (staging, >= 20 KiB)
  int rpp, passes;     // filter rows per pass, passes per tile (last may be shorter)
  int pstages;         // stages of a full pass: rpp * chunks <= kDcMaxStages
  int cw;              // channels per halo box (16 or 32)
  int halo_w;          // 3 * ow + 32 pixels
  int box_bytes;       // one halo box (rpp x halo_w x cw floats), 1 KiB aligned
  int slot_bytes;      // (c / cw) boxes
  int n_slots;         // halo ring depth
  int bbox;            // one filter stage box: n rows x 64 B
  int bres_bytes;      // resident filters, hi (same again for lo)
  int a_slots, a_cols; // TMEM A ring: slots of a_cols = pstages * 32 columns
  int n_part;          // TMEM accumulators (n columns each)
  uint32_t idesc;
  float alpha, beta;
  float* Y;
  unsigned long long* stats;  // debug (TM_CONV_STATS): [grid][16] cycles per role and wait, or null
};

// Role timing for TM_CONV_STATS (null stats: no cost beyond the branch).
enum DcStat { kStMmaWaitAcc, kStMmaWaitReady, kStMmaTotal, kStSplitWaitHalo, kStSplitWaitSlot, kStSplitTotal,
              kStEpiWaitAcc, kStEpiTotal, kStProdWaitSlot, kStProdTotal, kStMmaIssue, kStMmaCommit, kStMmaLoop, kStMmaFence, kStMmaBody };
#define DC_TIMED(slot, stmt)                                      \
  do {                                                            \
    if constexpr (ST) {                                           \
      const long long t0_ = clock64();                            \
      stmt;                                                       \
      st_acc[slot] += static_cast<unsigned long long>(clock64() - t0_); \
    } else {                                                      \
      stmt;                                                       \
    }                                                             \
  } while (0)

// Tile t -> image b, first output row y (ro rows per tile), first output column x0.
template <int RO>
__device__ __forceinline__ void dc_tile(const DcParams& p, int t, int& b, int& y, int& x0) {
  const int xt = t % p.tiles_x;
  const int rest = t / p.tiles_x;
  y = (rest % p.ho_t) * RO;
  b = rest / p.ho_t;
  x0 = xt * 4 * p.ow;
}

// RO: output rows per tile (== p.ro; a template parameter so that the one-row
// kernels, whose epilogue is the longer chain at wide filters, carry no loop).
template <int S, bool ST = false, int RO = 1>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_direct(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, DcParams p) {
  extern __shared__ uint8_t smem_raw_[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_) + 1023) & ~uintptr_t(1023));
  uint8_t* bres = smem;
  uint8_t* bres_lo = bres + p.bres_bytes;
  uint8_t* halo = bres_lo + p.bres_bytes;
  uint8_t* fstage = halo + p.n_slots * p.slot_bytes;  // ro == 2: raw filter boxes before expansion
  uint64_t* bres_full = reinterpret_cast<uint64_t*>(fstage + p.fgap);
  uint64_t* halo_full = bres_full + 1;            // [n_slots] TMA landed
  uint64_t* halo_empty = halo_full + p.n_slots;   // [n_slots] split warps done reading
  uint64_t* ready = halo_empty + p.n_slots;       // [kDcMaxSlots] A slot written
  uint64_t* a_empty = ready + kDcMaxSlots;        // [kDcMaxSlots] MMAs done with the slot (commit)
  uint64_t* part_full = a_empty + kDcMaxSlots;    // [2] accumulator complete (commit)
  uint64_t* part_empty = part_full + 2;           // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(part_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long st_acc[ST ? 16 : 1] = {};
  const long long st_t0 = ST ? clock64() : 0;
  (void)st_acc;
  (void)st_t0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bres_full, 1);
    for (int i = 0; i < p.n_slots; ++i) {
      ptx::mbar_init(&halo_full[i], 1);
      ptx::mbar_init(&halo_empty[i], kDcSplitWarps);
    }
    for (int i = 0; i < kDcMaxSlots; ++i) {
      ptx::mbar_init(&ready[i], kDcSplitWarps);
      ptx::mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&part_full[i], 1);
      ptx::mbar_init(&part_empty[i], kDcEpiWarps / 2);  // the accumulator's epilogue group
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmW);
  }
  if (warp == 2) ptx::tmem_alloc<1>(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t acol = static_cast<uint32_t>(p.n_part * p.n);  // first TMEM column of the A slots

  if (warp < 4) {
    ptx::setmaxnreg_dec<80>();
    if (warp == 0 || warp == 2) {
      // ------------------------------------------------------------ producers
      const int pi = warp >> 1;
      if (ptx::elect_one()) {
        if (pi == 0) {
          // filters: stage (ky, ci) = box {16 channels, S taps, 1, fp filters}
          // -> rows (f, kx) x 64 B, i.e. B^T of the Z GEMM for this K block
          // (ro == 2: into the staging area; the split warps expand them)
          uint8_t* fdst = RO == 2 ? fstage : bres;
          ptx::mbar_arrive_expect_tx(bres_full, static_cast<uint32_t>(p.fstages * p.fbox));
          for (int s = 0; s < p.fstages; ++s) {
            const int ky = s / p.chunks, ci = s - ky * p.chunks;
            ptx::tma_load_4d(fdst + s * p.fbox, &tmW, bres_full, ci * kDcBK, 0, p.kx0, ky);
          }
        }
        int slot = 0, own = 0;
        uint32_t ph = 0;
        const int boxes = p.c / p.cw;
        for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x)
        for (int ps = 0; ps < p.passes; ++ps) {
          if (own == pi) {
            int b, y, x0;
            dc_tile<RO>(p, t, b, y, x0);
            DC_TIMED(kStProdWaitSlot, ptx::mbar_wait(&halo_empty[slot], ph ^ 1));
            ptx::mbar_arrive_expect_tx(&halo_full[slot], static_cast<uint32_t>(boxes * p.rpp * p.halo_w * p.cw * 4));
            for (int i = 0; i < boxes; ++i)
              ptx::tma_load_4d(halo + slot * p.slot_bytes + i * p.box_bytes, &tmX, &halo_full[slot], i * p.cw,
                               x0 - p.pad, y - p.pad + ps * p.rpp, b);
            if (p.beta != 0.0f && ps == 0) {
              // the epilogue will read beta * Y for this tile's outputs (one
              // contiguous run of the output row): stage it in L2 now, the
              // halo ring depth ahead of its use
              const int cnt = min(4 * p.ow, p.wo - x0);
              for (int o = 0; o < RO && y + o < p.ho; ++o)
                ptx::prefetch_l2_bulk(p.Y + static_cast<long long>((b * p.ho + y + o) * p.wo + x0) * p.f,
                                      static_cast<uint32_t>(cnt * p.f * 4));
            }
          }
          if (++own == kDcProducers) own = 0;
          if (++slot == p.n_slots) { slot = 0; ph ^= 1; }
        }
      }
    } else if (warp == 1 && ptx::elect_one()) {
      // ------------------------------------------------------------ MMA issuer
      const uint32_t idesc = p.idesc;
      // descriptors advance by (bytes >> 4) in their start-address field
      const uint64_t bH0 = ptx::sdesc(ptx::smem_u32(bres), 16, 512, ptx::kLayoutSW64);
      const uint64_t bL0 = ptx::sdesc(ptx::smem_u32(bres_lo), 16, 512, ptx::kLayoutSW64);
      const uint32_t bstep = static_cast<uint32_t>(p.bbox >> 4);
      int sl = 0, pb = 0;
      uint32_t phl = 0, pph = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const long long tb0_ = ST ? clock64() : 0;
        DC_TIMED(kStMmaWaitAcc, ptx::mbar_wait(&part_empty[pb], pph ^ 1));
        const uint32_t d = tmem_base + static_cast<uint32_t>(pb * p.n);
        uint32_t boff = 0;
        int sg = 0;  // filter stage (global over the passes)
        for (int ps = 0; ps < p.passes; ++ps) {
          DC_TIMED(kStMmaWaitReady, ptx::mbar_wait(&ready[sl], phl));
          DC_TIMED(kStMmaFence, ptx::tc_fence_after());
          uint32_t a = tmem_base + acol + static_cast<uint32_t>(sl * p.a_cols);
          const int ns = min(p.pstages, p.stages - sg);
          const long long ti0_ = ST ? clock64() : 0;
          for (int s = 0; s < ns; ++s, ++sg) {
#pragma unroll
            for (int ks = 0; ks < kDcBK / 8; ++ks) {
              const uint64_t bH = bH0 + boff + 2 * ks, bL = bL0 + boff + 2 * ks;  // +32 B per K step of 8
              ptx::mma_tf32_tmem_a<1>(d, a + kDcBK + 8 * ks, bH, idesc, (sg | ks) ? 1u : 0u);  // A_lo B_hi
              ptx::mma_tf32_tmem_a<1>(d, a + 8 * ks, bL, idesc, 1u);                          // A_hi B_lo
              ptx::mma_tf32_tmem_a<1>(d, a + 8 * ks, bH, idesc, 1u);                          // A_hi B_hi
            }
            a += 2 * kDcBK;
            boff += bstep;
          }
          ptx::mma_commit<1>(&a_empty[sl]);
          if constexpr (ST) st_acc[kStMmaIssue] += static_cast<unsigned long long>(clock64() - ti0_);
          if (++sl == p.a_slots) { sl = 0; phl ^= 1; }
        }
        DC_TIMED(kStMmaCommit, ptx::mma_commit<1>(&part_full[pb]));
        if (++pb == p.n_part) { pb = 0; pph ^= 1; }
        if constexpr (ST) { st_acc[kStMmaLoop] += 1; st_acc[kStMmaBody] += static_cast<unsigned long long>(clock64() - tb0_); }
      }
    }
  } else if (warp < 8) {
    // -------------------------------------------------------------- split
    // keeps the launch's 128 registers: (80 + 128) * 128 + 152 * 256 = 65536
    const int q = warp & 3;
    {
      // resident filters: lo = split of hi, same layout (elementwise)
      const int st = q * 32 + lane;
      ptx::mbar_wait(bres_full, 0);
      if constexpr (RO == 2) {
        // Expand the raw boxes (rows (kx, f) of filter row ky) into the two-row
        // B^T: stage (input row j, channels ci), row (o, kx, f) = W[f, j - o, kx, c]
        // when 0 <= j - o < r, else zero.  16-B chunks through the SWIZZLE_64B
        // pattern of both layouts (chunk c of row r at c ^ ((r / 2) % 4); boxes
        // 1 KiB aligned).
        const uint32_t fs = ptx::smem_u32(fstage), bd = ptx::smem_u32(bres);
        const int per_stage = p.n * 4;  // 16-B chunks per expanded stage
        for (int i = st; i < p.stages * per_stage; i += 128) {
          const int sg = i / per_stage, rem = i - sg * per_stage;
          const int rr = rem >> 2, c = rem & 3;
          const int j = sg / p.chunks, ci = sg - j * p.chunks;
          const int o = rr / p.nrow, qrow = rr - o * p.nrow, ky = j - o;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (ky >= 0 && ky < p.r)
            v = ptx::lds128(fs + (ky * p.chunks + ci) * p.fbox + qrow * 64 + ((c ^ ((qrow >> 1) & 3)) << 4));
          ptx::sts128(bd + sg * p.bbox + rr * 64 + ((c ^ ((rr >> 1) & 3)) << 4), v);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // split warpgroup: expansion done before the lo pass
      }
      const uint32_t src = ptx::smem_u32(bres), dst = ptx::smem_u32(bres_lo);
      for (int i = st; i < p.bres_bytes / 16; i += 128) ptx::sts128(dst + i * 16, tf32_lo4(ptx::lds128(src + i * 16)));
      ptx::fence_proxy_async_smem();
    }
    const uint32_t halo_s = ptx::smem_u32(halo);
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acol;
    const bool cw16 = p.cw == 16;  // 64-B halo rows (SWIZZLE_64B), else 128-B rows (SWIZZLE_128B)
    const int rb = p.cw * 4;
    const int hp = p.ow * q + lane;  // this lane's halo pixel
    // Per-stage shared-memory offsets of this lane's 16 channels inside a halo
    // slot (tile-independent): stage s = (ky, 16-channel chunk ci).  TMA
    // swizzle (box bases 1 KiB aligned): 16-B chunk j of a row is stored at
    // j ^ ((row / 2) % 4) for 64-B rows, j ^ (row % 8) for 128-B rows.
    uint32_t soff[kDcMaxStages], sxor[kDcMaxStages];
#pragma unroll
    for (int s = 0; s < kDcMaxStages; ++s) {
      const int ky = s / p.chunks, ci = s - ky * p.chunks;  // row within the pass
      const int box = cw16 ? ci : (ci >> 1);
      const int within = cw16 ? 0 : ((ci & 1) << 2);  // first 16-B chunk of these 16 channels
      const int row = ky * p.halo_w + hp;             // pixel row inside the box
      soff[s] = static_cast<uint32_t>(box * p.box_bytes + row * rb);
      sxor[s] = static_cast<uint32_t>(cw16 ? ((row >> 1) & 3) : (row & 7));
      sxor[s] = (sxor[s] ^ static_cast<uint32_t>(within)) & 7u;  // within in {0, 4} and j < 4: (within + j) ^ sw = (j ^ (sw ^ within))
    }
    int slot = 0, sl = 0;
    uint32_t ph = 0, phl = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x)
    for (int ps = 0; ps < p.passes; ++ps) {
      {
        const int ns = min(p.pstages, p.stages - ps * p.pstages);
        DC_TIMED(kStSplitWaitHalo, ptx::mbar_wait(&halo_full[slot], ph));
        DC_TIMED(kStSplitWaitSlot, ptx::mbar_wait(&a_empty[sl], phl ^ 1));
        ptx::tc_fence_after();
        const uint32_t hb = halo_s + slot * p.slot_bytes;
        const uint32_t ta = trow + static_cast<uint32_t>(sl * p.a_cols);
#pragma unroll
        for (int s = 0; s < kDcMaxStages; ++s) {
          if (s >= ns) break;
          const uint32_t rowp = hb + soff[s];
          uint4 v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = ptx::lds128(rowp + ((static_cast<uint32_t>(j) ^ sxor[s]) << 4));
          uint32_t hl[32];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t x[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              hl[4 * j + e] = x[e];                           // A_hi: kind::tf32 truncates the raw value
              // A_lo = x - hi, exact in fp32, left for the tensor core to truncate
              // (2 ops instead of the RNA rounding's 4: this split warp is the
              // kernel's critical role; bound 5 * 2^-21 per product, reading 4)
              hl[kDcBK + 4 * j + e] = __float_as_uint(__fsub_rn(__uint_as_float(x[e]), __uint_as_float(x[e] & 0xFFFFE000u)));
            }
          }
          ptx::tmem_st_32x32b_x32(ta + s * 2 * kDcBK, hl);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&ready[sl]);
          ptx::mbar_arrive(&halo_empty[slot]);
        }
      }
      if (++slot == p.n_slots) { slot = 0; ph ^= 1; }
      if (++sl == p.a_slots) { sl = 0; phl ^= 1; }
    }
  } else {
    // -------------------------------------------------------------- promotion, shift-add, epilogue
    // Group e (warps 8-11, 12-15) drains accumulator e: with two accumulators
    // the groups alternate tiles, with one only group 0 works.
    ptx::setmaxnreg_inc<152>();
    const int q = warp & 3;
    const int e = (warp - 8) >> 2;
    const int pb = e;
    uint32_t pph = 0;
    int i = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++i) {
      if (i % p.n_part != e) continue;
      DC_TIMED(kStEpiWaitAcc, ptx::mbar_wait(&part_full[pb], pph));
      ptx::tc_fence_after();
      int b, y, x0;
      dc_tile<RO>(p, t, b, y, x0);
      const int xw = x0 + p.ow * q;                        // first output pixel of this warp
      const int valid = min(p.ow, p.wo - xw);              // outputs of this warp (lanes 0 .. valid-1)
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(pb * p.n);
      // ro output rows per tile: row o's Z columns start at o * nrow
#pragma unroll
      for (int o = 0; o < RO; ++o)
      for (int f0 = 0; f0 < p.fp; f0 += 16) {
        const int row0 = (b * p.ho + y + o) * p.wo + xw;   // this warp's first GEMM row (output pixel)
        const bool row_ok = y + o < p.ho;                  // the last tile row of an odd ho has one row
        const uint32_t taddr = tacc + static_cast<uint32_t>(o * p.nrow);
        // column kx * fp + f holds Z[., (f, kx)]: per kx, 16 consecutive columns
        // of filters f0 .. f0 + 15; loads in groups of KG taps (registers)
        constexpr int KG = S <= 7 ? S : (S + 1) / 2;
        float acc[16];
#pragma unroll
        for (int k0 = 0; k0 < S; k0 += KG) {
          uint32_t r[16 * KG];
#pragma unroll
          for (int c = 0; c < KG; ++c)
            if (k0 + c < S)
              ptx::tmem_ld_32x32b_x16(taddr + (k0 + c) * p.fp + f0, *reinterpret_cast<uint32_t(*)[16]>(r + 16 * c));
          ptx::tmem_ld_wait();
          if (o + 1 == RO && f0 + 16 >= p.fp && k0 + KG >= S) {  // last read of this accumulator: hand it back
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&part_empty[pb]);
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int c = 0; c < KG; ++c) {
              const int kx = k0 + c;
              if (kx >= S) continue;
              // tap p.kx0 + kx of output lane x sits in halo lane x + p.kx0 + kx
              const float z = __shfl_down_sync(0xffffffffu, __uint_as_float(r[16 * c + j]), p.kx0 + kx);
              if (kx == 0) acc[j] = z;  // first tap, then kx ascending
              else acc[j] += z;
            }
          }
        }
        // Output pixel row0 + lane owns Y[.., f0 .. f0 + 15]: 16 contiguous
        // floats (NHWC), so each lane stores its own float4s -- a warp's 30
        // pixels are one contiguous run of Y, completed in L2 by the four
        // stores -- with no shared-memory transpose (the GEMM epilogue's
        // staging cost bank conflicts here).  F % 4 == 0 (tensor-core rule).
        if (row_ok && lane < valid && f0 < p.f) {
          float* yp = p.Y + static_cast<long long>(row0 + lane) * p.f + f0;
          const int nf = min(16, p.f - f0);
          float4 cv[4];
#pragma unroll
          for (int v = 0; v < 4; ++v)
            cv[v] = (p.beta != 0.0f && 4 * v < nf) ? *reinterpret_cast<const float4*>(yp + 4 * v)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            if (4 * v >= nf) continue;
            float4 o;
            if (p.beta == 0.0f) {
              o = make_float4(p.alpha * acc[4 * v], p.alpha * acc[4 * v + 1], p.alpha * acc[4 * v + 2],
                              p.alpha * acc[4 * v + 3]);
            } else {
              o = make_float4(fmaf(p.alpha, acc[4 * v], p.beta * cv[v].x), fmaf(p.alpha, acc[4 * v + 1], p.beta * cv[v].y),
                              fmaf(p.alpha, acc[4 * v + 2], p.beta * cv[v].z), fmaf(p.alpha, acc[4 * v + 3], p.beta * cv[v].w));
            }
            *reinterpret_cast<float4*>(yp + 4 * v) = o;
          }
        }
      }
      pph ^= 1;
    }
  }

  if constexpr (ST) {  // one representative thread per role: producer 0, MMA, split warp 4, epilogue warp 8
    const unsigned long long total = static_cast<unsigned long long>(clock64() - st_t0);
    unsigned long long* o = p.stats + static_cast<long long>(blockIdx.x) * 16;
    if (threadIdx.x == 0) { o[kStProdWaitSlot] = st_acc[kStProdWaitSlot]; o[kStProdTotal] = total; }
    if (warp == 1 && lane == 0) { o[kStMmaWaitAcc] = st_acc[kStMmaWaitAcc]; o[kStMmaWaitReady] = st_acc[kStMmaWaitReady]; o[kStMmaTotal] = total; o[kStMmaIssue] = st_acc[kStMmaIssue]; o[kStMmaCommit] = st_acc[kStMmaCommit]; o[kStMmaLoop] = st_acc[kStMmaLoop]; o[kStMmaFence] = st_acc[kStMmaFence]; o[kStMmaBody] = st_acc[kStMmaBody]; }
    if (warp == 4 && lane == 0) { o[kStSplitWaitHalo] = st_acc[kStSplitWaitHalo]; o[kStSplitWaitSlot] = st_acc[kStSplitWaitSlot]; o[kStSplitTotal] = total; }
    if (warp == 8 && lane == 0) { o[kStEpiWaitAcc] = st_acc[kStEpiWaitAcc]; o[kStEpiTotal] = total; }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem_base, 512);
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

// KRSC filters as {C, F, S, R} (strides of the KRSC tensor reordered), box
// {16, fp, taps, 1}: rows (kx, f) of one (ky, 16 channels) stage -- B^T row
// (kx - kx0) * fp + f for the launch's taps kx0 .. kx0 + taps - 1; filters
// f >= F are zero-filled.
bool encode_filters(CUtensorMap* map, const ConvArgs& a, int fp, int taps) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(a.c), static_cast<cuuint64_t>(a.f), static_cast<cuuint64_t>(a.s),
                        static_cast<cuuint64_t>(a.r)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(a.c * a.s * a.r) * 4, static_cast<cuuint64_t>(a.c) * 4,
                           static_cast<cuuint64_t>(a.c * a.s) * 4};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(kDcBK), static_cast<cuuint32_t>(fp), static_cast<cuuint32_t>(taps), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(a.Wt), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Fills p and returns the dynamic shared-memory size, or 0 if the shape does
// not fit the direct kernel (then the implicit-GEMM kernel runs).  Passes:
// the largest RPP (filter rows per pass) for which two TMEM A slots fit beside
// the accumulators and the halo ring fits in shared memory, else the largest
// with one A slot; the resident filters (all R*C/16 stages, hi and lo) must
// fit in any case -- 9x9 x 16 channels does (166 KB), 11x11 does not.
int dc_plan(const ConvArgs& a, DcParams& p, int kx0, int taps) {
  if (a.s > 32 - 8 || taps < 1 || taps > 9 || kx0 < 0 || kx0 + taps > a.s) return 0;
  if (a.c % kDcBK != 0 || a.f > 64 || a.r < 1) return 0;
  const int64_t ho = a.ho(), wo = a.wo();
  if (ho <= 0 || wo <= 0) return 0;
  p = DcParams{};
  p.nb = static_cast<int>(a.nb);
  p.h = static_cast<int>(a.h);
  p.w = static_cast<int>(a.w);
  p.c = static_cast<int>(a.c);
  p.f = static_cast<int>(a.f);
  p.r = static_cast<int>(a.r);
  p.pad = static_cast<int>(a.pad);
  p.ho = static_cast<int>(ho);
  p.wo = static_cast<int>(wo);
  p.fp = (p.f + 15) / 16 * 16;
  if (p.fp * taps > 256) return 0;
  p.ow = 33 - static_cast<int>(a.s);
  p.kx0 = kx0;
  p.tiles_x = static_cast<int>((wo + 4 * p.ow - 1) / (4 * p.ow));
  const int64_t tiles = a.nb * ((ho + 1) / 2 * 2) * p.tiles_x;  // bound for either ro (exact count below)
  if (tiles > INT32_MAX / 2 || a.nb * ho * wo > INT32_MAX / 2) return 0;
  (void)tiles;
  p.chunks = p.c / kDcBK;
  if (p.chunks > kDcMaxStages) return 0;
  // Two output rows per tile when one row's MMA N is small (<= 48): input rows
  // r + 1 instead of 2r, so the split reads and stores 2/3 of the rows per
  // output at 3x3 (measured 0.433 -> 0.388 ms, scripts/r02/conv_ro.sh) while
  // the MMAs do 4/3 the work (the (j, o) blocks with j - o outside [0, r) are
  // zeros; kind::tf32 with A in TMEM costs N/2 cycles at any N, DESIGN 7.12).
  static const int env_ro = [] { const char* e = std::getenv("TM_CONV_RO"); return e ? std::atoi(e) : 0; }();
  p.nrow = p.fp * taps;
  p.ro = (env_ro == 1 || p.r < 2 || 2 * p.nrow > 96) ? 1 : 2;
  if (env_ro == 2 && 2 * p.nrow <= 256 && p.r >= 2 && taps <= 3) p.ro = 2;  // two-row kernels: taps <= 3
  p.rin = p.r + p.ro - 1;
  p.n = p.ro * p.nrow;
  p.ho_t = (p.ho + p.ro - 1) / p.ro;
  p.fstages = p.r * p.chunks;
  p.fbox = p.nrow * kDcBK * 4;
  p.stages = p.rin * p.chunks;
  p.cw = p.c % 32 == 0 ? 32 : 16;
  p.halo_w = 3 * p.ow + 32;
  p.num_tiles = static_cast<int>(a.nb * p.ho_t * p.tiles_x);
  p.bbox = p.n * kDcBK * 4;
  p.bres_bytes = p.stages * p.bbox;
  // The region after the halo ring (the two-row kernel's filter staging) is at
  // least 20 KiB: measured A/B (scripts/r02/conv_ab5.sh), the 9x9 kernel runs
  // 2.05 ms with the barriers 20 KiB past the halo ring and 2.49 ms with them
  // right after it, at the same pipeline configuration (cause not isolated).
  p.fgap = std::max(p.ro == 2 ? p.fstages * p.fbox : 0, 20 * 1024);
  const int fixed = 1024 + 2 * p.bres_bytes + p.fgap + 512;
  if (fixed >= kDcMaxSmem) return 0;
  int best_rpp = 0, best_slots = 0, best_part = 0;
  // TM_CONV_RPP (tests / experiments): cap the filter rows per pass
  static const int env_rpp = [] { const char* e = std::getenv("TM_CONV_RPP"); return e ? std::atoi(e) : 0; }();
  for (int want_slots = 2; want_slots >= 1 && !best_rpp; --want_slots) {
    for (int rpp = std::min({p.rin, kDcMaxStages / p.chunks, env_rpp > 0 ? env_rpp : 1 << 20}); rpp >= 1; --rpp) {
      const int a_cols = rpp * p.chunks * 2 * kDcBK;
      int part = 2, slots = (512 - 2 * p.n) / a_cols;
      if (slots < want_slots) { part = 1; slots = (512 - p.n) / a_cols; }
      if (slots < want_slots) continue;
      const int box = (rpp * p.halo_w * p.cw * 4 + 1023) / 1024 * 1024;
      if ((kDcMaxSmem - fixed) / ((p.c / p.cw) * box) < 2) continue;
      best_rpp = rpp;
      best_slots = slots;
      best_part = part;
      break;
    }
  }
  if (!best_rpp) return 0;
  p.rpp = best_rpp;
  p.passes = (p.rin + p.rpp - 1) / p.rpp;
  p.pstages = p.rpp * p.chunks;
  p.a_cols = p.pstages * 2 * kDcBK;
  p.n_part = best_part;
  p.a_slots = best_slots > kDcMaxSlots ? kDcMaxSlots : best_slots;
  p.box_bytes = (p.rpp * p.halo_w * p.cw * 4 + 1023) / 1024 * 1024;
  p.slot_bytes = (p.c / p.cw) * p.box_bytes;
  p.idesc = ptx::idesc_tf32(kDcLanes, p.n, 0, 0);
  const int slots = (kDcMaxSmem - fixed) / p.slot_bytes;
  p.n_slots = slots < 4 ? (slots & ~1) : 4;  // even (see kDcProducers)
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.Y = a.Y;
  return fixed + p.n_slots * p.slot_bytes;
}

template <int S, int RO = 1>
tm_status launch_dc(const ConvArgs& a, const DcParams& p, int smem, int num_sms, cudaStream_t stream) {
  CUtensorMap tmX, tmW;
  if (!encode_halo(&tmX, a, p.cw, p.halo_w, p.rpp)) return TM_ERR_INTERNAL;
  if (!encode_filters(&tmW, a, p.fp, S)) return TM_ERR_INTERNAL;
  auto kern = k_conv_direct<S, false, RO>;
  static std::atomic<unsigned long long> optin{0};  // per instantiation, bit per device
  if (tm_status st = ensure_smem_optin(optin, kern, kDcMaxSmem); st != TM_OK) return st;
  const int grid = p.num_tiles < num_sms ? p.num_tiles : num_sms;
  const char* stats_path = std::getenv("TM_CONV_STATS");  // debug: per-role wait breakdown (scripts/r02/)
  if (!stats_path) {
    kern<<<grid, kThreads, smem, stream>>>(tmX, tmW, p);
    return cudaPeekAtLastError() == cudaSuccess ? TM_OK : TM_ERR_CUDA;
  }
  DcParams q = p;
  if (cudaMalloc(&q.stats, sizeof(unsigned long long) * 16 * grid) != cudaSuccess) return TM_ERR_CUDA;
  cudaMemsetAsync(q.stats, 0, sizeof(unsigned long long) * 16 * grid, stream);
  auto kst = k_conv_direct<S, true, RO>;
  static std::atomic<unsigned long long> optin_st{0};
  if (tm_status st = ensure_smem_optin(optin_st, kst, kDcMaxSmem); st != TM_OK) return st;
  kst<<<grid, kThreads, smem, stream>>>(tmX, tmW, q);
  if (cudaPeekAtLastError() != cudaSuccess) return TM_ERR_CUDA;
  std::vector<unsigned long long> h(16 * grid);
  cudaStreamSynchronize(stream);
  cudaMemcpy(h.data(), q.stats, sizeof(unsigned long long) * 16 * grid, cudaMemcpyDeviceToHost);
  cudaFree(q.stats);
  if (FILE* f = std::fopen(stats_path, "a")) {
    static const char* names[] = {"mma_wait_acc", "mma_wait_ready", "mma_total", "split_wait_halo", "split_wait_slot",
                                  "split_total", "epi_wait_acc", "epi_total", "prod_wait_slot", "prod_total", "mma_issue", "mma_commit", "mma_tiles", "mma_fence", "mma_body"};
    std::fprintf(f, "{\"S\": %d, \"tiles\": %d, \"grid\": %d", S, p.num_tiles, grid);
    for (int k = 0; k < 15; ++k) {
      double sum = 0;
      for (int b = 0; b < grid; ++b) sum += static_cast<double>(h[b * 16 + k]);
      std::fprintf(f, ", \"%s\": %.0f", names[k], sum / grid);
    }
    std::fprintf(f, "}\n");
    std::fclose(f);
  }
  return TM_OK;
}

}  // namespace

// The direct kernel takes the whole filter width in one launch when its
// resident filters fit; otherwise (11x11 x 16 channels: 248 KB of hi + lo
// filters) the filter columns are split in two launches, kx in [0, S1) and
// [S1, S): the second adds its taps to the first's result (beta = 1), at the
// cost of reading X twice and Y once more -- the tensor work, which bounds
// these shapes, is unchanged.
static bool dc_split(const ConvArgs& a, DcParams& p1, int& s1, DcParams& p2, int& s2, int& smem1, int& smem2) {
  s1 = static_cast<int>(a.s);
  s2 = 0;
  if ((smem1 = dc_plan(a, p1, 0, s1)) > 0) return true;
  s1 = static_cast<int>((a.s + 1) / 2);
  s2 = static_cast<int>(a.s) - s1;
  smem1 = dc_plan(a, p1, 0, s1);
  smem2 = dc_plan(a, p2, s1, s2);
  return smem1 > 0 && smem2 > 0;
}

int conv_direct_launches(const ConvArgs& a) {
  DcParams p1, p2;
  int s1, s2, m1, m2;
  if (!dc_split(a, p1, s1, p2, s2, m1, m2)) return 0;
  return s2 > 0 ? 2 : 1;
}

bool conv_direct_fits(const ConvArgs& a) { return conv_direct_launches(a) > 0; }

static tm_status launch_taps(const ConvArgs& a, const DcParams& p, int taps, int smem, int num_sms, cudaStream_t stream) {
  switch (taps) {
    case 1: return p.ro == 2 ? launch_dc<1, 2>(a, p, smem, num_sms, stream) : launch_dc<1>(a, p, smem, num_sms, stream);
    case 2: return p.ro == 2 ? launch_dc<2, 2>(a, p, smem, num_sms, stream) : launch_dc<2>(a, p, smem, num_sms, stream);
    case 3: return p.ro == 2 ? launch_dc<3, 2>(a, p, smem, num_sms, stream) : launch_dc<3>(a, p, smem, num_sms, stream);
    case 4: return launch_dc<4>(a, p, smem, num_sms, stream);
    case 5: return launch_dc<5>(a, p, smem, num_sms, stream);
    case 6: return launch_dc<6>(a, p, smem, num_sms, stream);
    case 7: return launch_dc<7>(a, p, smem, num_sms, stream);
    case 8: return launch_dc<8>(a, p, smem, num_sms, stream);
    case 9: return launch_dc<9>(a, p, smem, num_sms, stream);
    default: return TM_ERR_INVALID_VALUE;
  }
}

tm_status launch_conv_direct(const ConvArgs& a, int num_sms, cudaStream_t stream) {
  DcParams p1, p2;
  int s1, s2, m1, m2;
  if (!dc_split(a, p1, s1, p2, s2, m1, m2)) return TM_ERR_INVALID_VALUE;
  tm_status st = launch_taps(a, p1, s1, m1, num_sms, stream);
  if (st != TM_OK || s2 == 0) return st;
  p2.beta = 1.0f;  // add the remaining taps to the first launch's result
  return launch_taps(a, p2, s2, m2, num_sms, stream);
}

}  // namespace tmk
