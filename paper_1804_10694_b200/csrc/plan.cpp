// plan.cpp -- tile-configuration planner for the tensor-core path.
//
// The paper auto-tunes tile sizes for its sgemm; here the
// choice is a closed-form cost model over the compiled configurations:
// makespan = waves x per-tile MMA time / efficiency, where
//   tile      = (128*cg) x (bn*cg)            (CTA pair when cg == 2)
//   waves     = ceil(tiles / (num_sms / cg))  (persistent clusters)
//   per-tile  = ceil(k/32) * 4 K=8 steps * 3 MMAs * (cg*bn/2) cycles
//               (tcgen05 floor max(M,128)*N/(256*cg) with M = 128*cg, N = bn*cg)
//   efficiency: 1-CTA tiles read both operands from one SM's shared memory
//               (about 1.5x the smem bytes per MMA of a CTA pair), and narrow
//               tiles pay fixed per-stage costs -- measured factors, DESIGN.md.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "tm_internal.h"

namespace tmk {

// Stream-K pays off when the data-parallel schedule leaves a partial last
// wave that matters: fewer than 8 waves, tiles not a multiple of the cluster
// count, and at least 2 K-blocks of work per cluster.  Except for long-K
// schedules of >= 2 waves whose last wave is nearly full: data-parallel, they
// keep the clusters in step with the wave barrier (tc_gemm.cuh; L2 panel
// reuse), which stream-K cannot, and under the sustained power cap that is
// worth more than the partial wave: one rank of the 8-way row-sharded C5,
// 2048 x 16384 x 16384 = 512 tiles on 74 clusters (6.92 waves), runs in
// 4.01 ms data-parallel vs 4.70 ms stream-K (scripts/r02/rank_probe.py).
bool plan_streamk(int64_t m, int64_t n, int64_t k, int cg, int bn_cta, int num_sms) {
  const int64_t tile_m = 128LL * cg, tile_n = static_cast<int64_t>(bn_cta) * cg;
  const int64_t tiles = ((m + tile_m - 1) / tile_m) * ((n + tile_n - 1) / tile_n);
  const int64_t units = num_sms / cg;
  const int64_t kb = (k + 31) / 32;
  if (tiles % units == 0) return false;
  if (tiles >= 8 * units) return false;
  const int64_t waves = (tiles + units - 1) / units;
  const double wave_fill = static_cast<double>(tiles) / static_cast<double>(waves * units);
  if (kb >= 64 && tiles >= 2 * units && wave_fill >= 0.9) return false;
  return tiles * kb >= 2 * units;
}

// Stream-K region of a stream-K launch (tc_gemm.cuh launch_kernel; DESIGN 6.1
// "hybrid stream-K"): how many of the tiles are split over the clusters (the
// first sk_tiles of the raster; the rest run whole after each cluster's share)
// and how many clusters the launch uses.  mode: 0 pure stream-K, 1 the partial
// wave, 2 the partial wave plus one full wave, < 0 the default (2 for tiles of
// fewer than 64 K-blocks, else 1).  Invariants (tests/test_abi.py): every
// cluster owns at least two iterations of the region -- a finalizer waits for
// each later cluster whose range starts inside its tile, and an empty range
// would never publish -- and the tiles after the region form whole waves.
int64_t streamk_region(int64_t num_tiles, int64_t kblocks, int clusters, int mode, int* clusters_used) {
  if (mode < 0) mode = kblocks < 64 ? 2 : 1;
  int64_t sk = num_tiles;
  if (mode && num_tiles >= clusters) {
    sk = num_tiles % clusters;
    if (mode == 2 && num_tiles >= 2LL * clusters) sk += clusters;
    if (sk * kblocks < 2LL * clusters) sk = num_tiles;  // too few iterations: pure stream-K
  }
  const int64_t iters = sk * kblocks;
  if (sk == num_tiles && iters < 2LL * clusters) clusters = static_cast<int>(iters / 2 > 0 ? iters / 2 : 1);
  *clusters_used = clusters;
  return sk;
}

TcChoice plan_tc(int64_t m, int64_t n, int64_t k, int num_sms) {
  static const TcChoice cands[] = {{2, 128, 1, false}, {2, 64, 1, false}, {2, 32, 1, false},
                                   {1, 128, 1, false}, {1, 64, 1, false}, {1, 32, 1, false}};
  TcChoice best = cands[0];
  double best_t = 1e300;
  const int64_t kb = (k + 31) / 32;
  // Latency-bound one-wave problems (every 128 x 32 tile gets its own SM, short
  // K): the narrowest 1-CTA tile, data-parallel, has the least per-CTA work
  // between launch and epilogue -- the measured best from 128^3 to 768^3
  // (scripts/r02/small_probe.py, profiles/small_probe_r02.txt).
  if (((m + 127) / 128) * ((n + 31) / 32) <= num_sms && kb <= 32) return TcChoice{1, 32, 1, false};
  for (const TcChoice& c : cands) {
    const int64_t tile_m = 128LL * c.cg, tile_n = static_cast<int64_t>(c.bn_cta) * c.cg;
    const int64_t tiles = ((m + tile_m - 1) / tile_m) * ((n + tile_n - 1) / tile_n);
    const int64_t units = num_sms / c.cg;
    const int64_t waves = (tiles + units - 1) / units;
    const bool sk = plan_streamk(m, n, k, c.cg, c.bn_cta, num_sms);
    const double kb_cycles = 4.0 * 3.0 * (c.cg * c.bn_cta / 2.0);
    // + fixed per-tile cost: pipeline fill and the epilogue (about 5 us, ~10k
    // cycles, measured with TM_TRACE_PATH), scaled by the tile's column count
    const double epi = 4000.0 + 6000.0 * (c.cg * c.bn_cta) / 256.0;
    double per_tile = static_cast<double>(kb) * kb_cycles + epi;
    // Sustained MMA efficiency per configuration, measured on B200 at 8192^3
    // (DESIGN.md "Planner"): narrower tiles re-read A from shared memory more
    // often per MMA and a 1-CTA tile reads all of B from one SM.
    double eff = 1.0;
    if (c.cg == 2) eff = (c.bn_cta == 128) ? 1.0 : (c.bn_cta == 64) ? 0.88 : 0.58;
    else eff = (c.bn_cta == 128) ? 0.79 : (c.bn_cta == 64) ? 0.49 : 0.3;
    // Wasted MMA work on zero-filled tile padding is already in `waves`.
    double t = static_cast<double>(waves) * per_tile / eff;
    if (sk) {  // balanced iterations + one fixed-order reduction per cluster
      const double iters = static_cast<double>(tiles) * static_cast<double>(kb);
      // + one serial fixed-order reduction per tile over ~units/tiles partials
      const double parts = std::max(1.0, static_cast<double>(units) / static_cast<double>(tiles));
      t = (std::ceil(iters / static_cast<double>(units)) * kb_cycles + epi + parts * 3000.0 * (c.cg * c.bn_cta) / 256.0) /
          eff;
    }
    if (t < best_t * 0.999) {
      best_t = t;
      best = c;
      best.streamk = sk;
    }
  }
  return best;
}

}  // namespace tmk

extern "C" tm_status tm_sgemm_streamk_region(int64_t num_tiles, int64_t kblocks, int clusters, int mode,
                                             int64_t* sk_tiles, int* clusters_used) {
  if (num_tiles < 1 || kblocks < 1 || clusters < 1 || mode > 2 || !sk_tiles || !clusters_used)
    return TM_ERR_INVALID_VALUE;
  *sk_tiles = tmk::streamk_region(num_tiles, kblocks, clusters, mode, clusters_used);
  return TM_OK;
}
