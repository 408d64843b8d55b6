// Compile-time-shape building blocks for the specialized kernels: a "group"
// of NWG warps cooperates on one segment (NWG = 1 for n <= 16), synchronized
// with __syncwarp (NWG = 1) or a named barrier, so CTAs can hold several
// independent segments without CTA-wide barriers.
#pragma once

#include "plq_device.cuh"

#include <type_traits>

namespace plq {

// smallest v >= x with v % 8 == 4: row strides (in doubles) for which the
// DMMA fragment loads A[g][q] / B[q][g] (g = lane/4, q = lane%4) hit 16
// distinct 8-byte banks per half-warp, i.e. are shared-memory conflict-free
__host__ __device__ constexpr int pad_ld(int x) { return ((x + 3) / 8) * 8 + 4; }

static_assert(pad_ld(12) == 12 && pad_ld(17) == 20 && pad_ld(25) == 28 && pad_ld(32) == 36 && pad_ld(41) == 44 &&
                  pad_ld(65) == 68 && pad_ld(13) == 20 && pad_ld(4) == 4 && pad_ld(5) == 12,
              "pad_ld");

template <int NWG>
__device__ __forceinline__ void gsync(int grp) {
  if constexpr (NWG == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(NWG * 32) : "memory");
  }
}

// Group sum over NWG warps; `red` holds NWG doubles of this group's scratch.
template <int NWG>
__device__ __forceinline__ double gsum(double v, double* red, int grp, int gw) {
  v = warp_sum(v);
  if constexpr (NWG == 1) {
    return v;
  } else {
    gsync<NWG>(grp);
    if ((threadIdx.x & 31) == 0) red[gw] = v;
    gsync<NWG>(grp);
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NWG; ++w) t += red[w];
    return t;
  }
}

// Two group sums in one reduction pass (independent shuffle chains).
template <int NWG>
__device__ __forceinline__ double2 gsum2(double a, double b, double* red, int grp, int gw) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if constexpr (NWG == 1) {
    return make_double2(a, b);
  } else {
    gsync<NWG>(grp);
    if ((threadIdx.x & 31) == 0) {
      red[2 * gw] = a;
      red[2 * gw + 1] = b;
    }
    gsync<NWG>(grp);
    double ta = 0.0, tb = 0.0;
#pragma unroll
    for (int w = 0; w < NWG; ++w) {
      ta += red[2 * w];
      tb += red[2 * w + 1];
    }
    return make_double2(ta, tb);
  }
}

// C(M x N) = A (M x K) * B (K x N) on the FP64 tensor pipe (DMMA 8x8x4),
// compile-time shapes, operands supplied by loader functors aload(i, k) /
// bload(k, j) (only called in range).  Rows are processed in 8-row bands,
// band tm by warp (tm % NWG) of the group; `rows` <= M trims the bands at
// run time (constraint-row GEMMs).  With a single-warp group the band loop
// is unrolled so independent DMMA chains of different bands interleave.
// epi(i, j, acc) receives each element once.
template <int M, int N, int K, int NWG, class AL, class BL, class Epi>
__device__ __forceinline__ void ggemm_f(AL aload, BL bload, int gw, Epi epi, int rows = M) {
  constexpr int TM = (M + 7) / 8, TN = (N + 7) / 8, KS = (K + 3) / 4;
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  auto band = [&](int tm) {
    double acc[TN][2];
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) acc[tn][0] = acc[tn][1] = 0.0;
    const int i = tm * 8 + g;
    const bool iok = (i < M) && (i < rows);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = ks * 4 + q;
      const bool kok = (K % 4 == 0) || (k < K);
      const double a = (iok && kok) ? aload(i, k) : 0.0;
#pragma unroll
      for (int tn = 0; tn < TN; ++tn) {
        const int j = tn * 8 + g;
        const double b = (((N % 8 == 0) || (j < N)) && kok) ? bload(k, j) : 0.0;
        dmma884(acc[tn][0], acc[tn][1], a, b);
      }
    }
#pragma unroll
    for (int tn = 0; tn < TN; ++tn)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tn * 8 + 2 * q + e;
        if (iok && j < N) epi(i, j, acc[tn][e]);
      }
  };
  if constexpr (NWG == 1) {
    // single warp: every tile accumulated k-outer (one A fragment per band
    // and one B fragment per column tile per k-step, instead of reloading B
    // for every band), epilogue after all loads -- in-place safe
    double acc[TM][TN][2];
#pragma unroll
    for (int tm = 0; tm < TM; ++tm)
#pragma unroll
      for (int tn = 0; tn < TN; ++tn) acc[tm][tn][0] = acc[tm][tn][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = ks * 4 + q;
      const bool kok = (K % 4 == 0) || (k < K);
      double bv[TN];
#pragma unroll
      for (int tn = 0; tn < TN; ++tn) {
        const int j = tn * 8 + g;
        bv[tn] = (((N % 8 == 0) || (j < N)) && kok) ? bload(k, j) : 0.0;
      }
#pragma unroll
      for (int tm = 0; tm < TM; ++tm) {
        if (tm * 8 >= rows) continue;
        const int i = tm * 8 + g;
        const double a = ((i < M) && (i < rows) && kok) ? aload(i, k) : 0.0;
#pragma unroll
        for (int tn = 0; tn < TN; ++tn) dmma884(acc[tm][tn][0], acc[tm][tn][1], a, bv[tn]);
      }
    }
#pragma unroll
    for (int tm = 0; tm < TM; ++tm) {
      const int i = tm * 8 + g;
      if (tm * 8 >= rows || !(i < M && i < rows)) continue;
#pragma unroll
      for (int tn = 0; tn < TN; ++tn)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = tn * 8 + 2 * q + e;
          if (j < N) epi(i, j, acc[tm][tn][e]);
        }
    }
    (void)band;
  } else {
#pragma unroll 1
    for (int tm = gw; tm < TM; tm += NWG) {
      if (tm * 8 >= rows) break;
      band(tm);
    }
  }
}

// Same GEMM for single-warp groups with the epilogue also told the
// compile-time fragment slot (tm * TN + tn) * 2 + e, so per-element operands
// prefetched into a register array can be indexed statically.
template <int M, int N, int K, class AL, class BL, class Epi>
__device__ __forceinline__ void wgemm_slots(AL aload, BL bload, Epi epi) {
  constexpr int TM = (M + 7) / 8, TN = (N + 7) / 8, KS = (K + 3) / 4;
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  double acc[TM][TN][2];
#pragma unroll
  for (int tm = 0; tm < TM; ++tm)
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) acc[tm][tn][0] = acc[tm][tn][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + q;
    const bool kok = (K % 4 == 0) || (k < K);
    double bv[TN];
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) {
      const int j = tn * 8 + g;
      bv[tn] = (((N % 8 == 0) || (j < N)) && kok) ? bload(k, j) : 0.0;
    }
#pragma unroll
    for (int tm = 0; tm < TM; ++tm) {
      const int i = tm * 8 + g;
      const double a = ((i < M) && kok) ? aload(i, k) : 0.0;
#pragma unroll
      for (int tn = 0; tn < TN; ++tn) dmma884(acc[tm][tn][0], acc[tm][tn][1], a, bv[tn]);
    }
  }
#pragma unroll
  for (int tm = 0; tm < TM; ++tm) {
    const int i = tm * 8 + g;
#pragma unroll
    for (int tn = 0; tn < TN; ++tn)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tn * 8 + 2 * q + e;
        if (i < M && j < N) epi(i, j, acc[tm][tn][e], (tm * TN + tn) * 2 + e);
      }
  }
}

// Tile-selective group GEMM: warp gw processes the row bands bandof(gw, slot)
// (slot < NSLOT; a negative band is skipped) and, in band tm, only the 8 x 8
// column tiles with on(tm, tn) -- e.g. the lower triangle of a symmetric
// block, or no wasted blocks.  pre(i, j) is an addend (e.g. a Q-block entry
// read from global memory) loaded BEFORE the k-loop so its latency hides
// behind the DMMAs; epi(i, j, pre + acc) receives each selected element once.
template <int M, int N, int K, int NSLOT, class BandOf, class On, class AL, class BL, class Pre, class Epi>
__device__ __forceinline__ void ggemm_sel(AL aload, BL bload, int gw, BandOf bandof, On on, Pre pre, Epi epi) {
  constexpr int TN = (N + 7) / 8, KS = (K + 3) / 4;
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
#pragma unroll 1
  for (int slot = 0; slot < NSLOT; ++slot) {
    const int tm = bandof(gw, slot);
    if (tm < 0) continue;
    const int i = tm * 8 + g;
    const bool iok = i < M;
    double acc[TN][2], add[TN][2];
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) {
      acc[tn][0] = acc[tn][1] = 0.0;
      add[tn][0] = add[tn][1] = 0.0;
      if (on(tm, tn)) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = tn * 8 + 2 * q + e;
          if (iok && j < N) add[tn][e] = pre(i, j);
        }
      }
    }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = ks * 4 + q;
      const bool kok = (K % 4 == 0) || (k < K);
      const double a = (iok && kok) ? aload(i, k) : 0.0;
#pragma unroll
      for (int tn = 0; tn < TN; ++tn) {
        if (on(tm, tn)) {
          const int j = tn * 8 + g;
          const double b = (((N % 8 == 0) || (j < N)) && kok) ? bload(k, j) : 0.0;
          dmma884(acc[tn][0], acc[tn][1], a, b);
        }
      }
    }
#pragma unroll
    for (int tn = 0; tn < TN; ++tn) {
      if (on(tm, tn)) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = tn * 8 + 2 * q + e;
          if (iok && j < N) epi(i, j, add[tn][e] + acc[tn][e]);
        }
      }
    }
  }
}

// Two row bands of a tile-selective GEMM in ONE k-loop: band tmA (column
// tiles tn < TNA with on(tmA, tn)) and band tmB (tn < TNB with on(tmB, tn);
// tmB < 0: band A only).  Every k-step issues the DMMAs of both bands' tiles
// back to back, so a band with few tiles (the short end of a triangular
// block) no longer runs its K/4-deep accumulation chain alone.  Addends:
// pre(i, j) is loaded before the k-loop for every band-A tile when PREA and
// for the band-B tiles tn >= PRE_FROM (latency hidden behind the DMMAs);
// epi(i, j, v, has_pre) gets v = pre + acc for those and v = acc otherwise
// (the epilogue then adds its on-chip addend itself, which keeps the
// register footprint down).
// The bands are template parameters (tmA, tmB; tmB < 0: none) so that, once
// the tile loops are unrolled, on(tm, tn) folds to a constant: no runtime
// tile predicates in the k-loop (callers dispatch on the warp index).
template <int M, int N, int K, int TNA, int TNB, bool PREA, int PRE_FROM, int tmA, int tmB, class AL, class BL,
          class On, class Pre, class Epi>
__device__ __forceinline__ void ggemm_sel2(AL aload, BL bload, On on, Pre pre, Epi epi) {
  constexpr int KS = (K + 3) / 4;
  constexpr int TNX = TNA > TNB ? TNA : TNB;
  constexpr int TPA = PREA ? TNA : 1, TPB = TNB > PRE_FROM ? TNB - PRE_FROM : 1;
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int iA = tmA * 8 + g, iB = tmB * 8 + g;
  constexpr bool hasB = tmB >= 0;
  const bool okA = iA < M, okB = hasB && iB < M;
  double accA[TNA][2], accB[TNB > 0 ? TNB : 1][2], addA[TPA][2], addB[TPB][2];
#pragma unroll
  for (int tn = 0; tn < TNA; ++tn) accA[tn][0] = accA[tn][1] = 0.0;
#pragma unroll
  for (int tn = 0; tn < TNB; ++tn) accB[tn][0] = accB[tn][1] = 0.0;
  if constexpr (PREA) {
#pragma unroll
    for (int tn = 0; tn < TNA; ++tn)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tn * 8 + 2 * q + e;
        addA[tn][e] = (okA && j < N && on(tmA, tn)) ? pre(iA, j) : 0.0;
      }
  }
#pragma unroll
  for (int tn = PRE_FROM; tn < TNB; ++tn)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = tn * 8 + 2 * q + e;
      addB[tn - PRE_FROM][e] = (okB && j < N && on(tmB, tn)) ? pre(iB, j) : 0.0;
    }
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + q;
    const bool kok = (K % 4 == 0) || (k < K);
    const double a = (okA && kok) ? aload(iA, k) : 0.0;
    const double ab = (okB && kok) ? aload(iB, k) : 0.0;
#pragma unroll
    for (int tn = 0; tn < TNX; ++tn) {
      const int j = tn * 8 + g;
      const bool useA = tn < TNA && on(tmA, tn), useB = tn < TNB && hasB && on(tmB, tn);
      if (useA || useB) {
        const double b = (((N % 8 == 0) || (j < N)) && kok) ? bload(k, j) : 0.0;
        if (tn < TNA && useA) dmma884(accA[tn < TNA ? tn : 0][0], accA[tn < TNA ? tn : 0][1], a, b);
        if (tn < TNB && useB) dmma884(accB[tn < TNB ? tn : 0][0], accB[tn < TNB ? tn : 0][1], ab, b);
      }
    }
  }
#pragma unroll
  for (int tn = 0; tn < TNA; ++tn) {
    if (on(tmA, tn)) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tn * 8 + 2 * q + e;
        if (okA && j < N) epi(iA, j, accA[tn][e] + (PREA ? addA[PREA ? tn : 0][e] : 0.0), PREA);
      }
    }
  }
#pragma unroll
  for (int tn = 0; tn < TNB; ++tn) {
    if (hasB && on(tmB, tn)) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tn * 8 + 2 * q + e;
        const bool hp = tn >= PRE_FROM;
        if (okB && j < N) epi(iB, j, accB[tn][e] + (hp ? addB[hp ? tn - PRE_FROM : 0][e] : 0.0), hp);
      }
    }
  }
}

// f(std::integral_constant<int, w>{}) for the runtime warp index w < 8:
// lets a group hand each warp a compile-time role.
template <class F>
__device__ __forceinline__ void warp_dispatch8(int w, F&& f) {
  switch (w) {
    case 0: f(std::integral_constant<int, 0>{}); break;
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    default: f(std::integral_constant<int, 7>{}); break;
  }
}

// pointer-operand form: A row-major (or transposed, TA) with stride LDA, B row-major stride LDB
template <int M, int N, int K, bool TA, int LDA, int LDB, int NWG, class Epi>
__device__ __forceinline__ void ggemm(const double* __restrict__ A, const double* __restrict__ B, int gw, Epi epi,
                                      int rows = M) {
  ggemm_f<M, N, K, NWG>([&](int i, int k) { return TA ? A[k * LDA + i] : A[i * LDA + k]; },
                        [&](int k, int j) { return B[k * LDB + j]; }, gw, epi, rows);
}

}  // namespace plq
