// K1 host side: CTA size, shared-memory / scratch layout and the launch
// dispatch over the per-CTA-size instantiations (plq_sweep_t<NT>.cu, kernel
// body in plq_sweep_impl.cuh).
#include "plq_gemm.cuh"
#include "plq_internal.h"

#include <algorithm>

namespace plq {

#define PLQ_SWEEP_DECLARE(NT)                                                    \
  int launch_sweep_##NT(const SweepArgs& a, int grid, size_t smem, cudaStream_t s); \
  int launch_sweep_repair_##NT(const SweepArgs& a, int grid, size_t smem, cudaStream_t s); \
  int sweep_occupancy_##NT(size_t smem);
PLQ_SWEEP_DECLARE(32)
PLQ_SWEEP_DECLARE(128)
PLQ_SWEEP_DECLARE(256)
PLQ_SWEEP_DECLARE(512)

int sweep_threads(int n) {
  if (n <= 16) return 32;
  if (n <= 32) return 128;
  // n > 32: 8-warp CTAs, two per SM (128 registers each); at n = 128 (cfg3)
  // this keeps all 256 segments resident at once, so one segment's serial
  // phases overlap the other's GEMMs (20.5 vs 25.0 ms sweep with 16-warp CTAs)
  return 256;
}

SweepLayout plan_sweep(int n, int m, int threads, size_t smem_budget) {
  // storage strides (even in large mode, see sweep_segment)
  const bool large = n >= 48;
  const int64_t Fw = large ? ((n + m + 2) & ~1) : n + m + 1, W = large ? 2 * n + 2 : 2 * n + 1;
  int64_t sz[SB_COUNT];
  sz[SB_V] = 3LL * n * n + 2 * n;
  sz[SB_IN] = n * Fw + (int64_t)n * n + (int64_t)m * n + (int64_t)m * m + n + m;
  sz[SB_PGY] = 3 * m * W;
  sz[SB_MUU] = 2LL * m * m;
  // tau, rdiag, reduction (32), flags (2), blocked scratch: block inverses,
  // per-warp tiles, V T' (plq_blocked.cuh)
  sz[SB_MISC] = 2LL * m + 32 + 2 + ((m + 7) / 8) * 64LL + (threads / 32) * 64LL + 16LL * n + 64 +
                (sweep_muu_in_smem(n, m) ? (int64_t)m * (m + 4) + 2 : 0);
  sz[SB_VF] = n * Fw;
  sz[SB_Z] = n * Fw;
  sz[SB_MX] = 0;   // Mxx / mx1 are written into Vxx / vx1 in place
  sz[SB_H] = n * W;
  const bool wide = (n % m) != 0;
  sz[SB_WIDE] = wide ? ((int64_t)m * std::min(n, m) + (int64_t)m * m + 2 * m * W) : 0;
  SweepLayout L{};
  int64_t so = 0, go = 0;
  int64_t budget = (int64_t)(smem_budget / sizeof(double));
  if (n >= 48) {
    // large mode: GEMM operands stay in (L2-resident) global scratch and are
    // streamed through shared-memory tiles; only MISC lives in smem
    L.large = 1;
    const int nw = threads / 32;
    L.tiles_off = 0;
    so = nw >= 16 ? TileCfg<16, sweep_tile_stages(512)>::DOUBLES
                  : (nw >= 8 ? TileCfg<8, sweep_tile_stages(256)>::DOUBLES : TileCfg<4>::DOUBLES);
    budget = so + ((sz[SB_MISC] + 1) & ~1LL);
  }
  for (int i = 0; i < SB_COUNT; ++i) {
    const int64_t s = (sz[i] + 1) & ~1LL;   // 16-byte granules
    if (i == SB_MISC || (!L.large && so + s <= budget)) {
      L.off[i] = so;
      L.in_smem[i] = 1;
      so += s;
    } else {
      L.off[i] = go;
      L.in_smem[i] = 0;
      go += s;
    }
  }
  L.smem_doubles = so;
  L.gmem_doubles = go;
  return L;
}

int launch_sweep(const SweepArgs& a, int grid, int threads, size_t smem, cudaStream_t s) {
  if (a.repair) {
    switch (threads) {
      case 32: return launch_sweep_repair_32(a, grid, smem, s);
      case 128: return launch_sweep_repair_128(a, grid, smem, s);
      case 256: return launch_sweep_repair_256(a, grid, smem, s);
      default: return launch_sweep_repair_512(a, grid, smem, s);
    }
  }
  switch (threads) {
    case 32: return launch_sweep_32(a, grid, smem, s);
    case 128: return launch_sweep_128(a, grid, smem, s);
    case 256: return launch_sweep_256(a, grid, smem, s);
    default: return launch_sweep_512(a, grid, smem, s);
  }
}

// Occupancy helper used by the C-ABI layer to size the persistent grid.
int sweep_max_blocks_per_sm(int threads, size_t smem) {
  switch (threads) {
    case 32: return sweep_occupancy_32(smem);
    case 128: return sweep_occupancy_128(smem);
    case 256: return sweep_occupancy_256(smem);
    default: return sweep_occupancy_512(smem);
  }
}

}  // namespace plq
