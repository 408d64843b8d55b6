// Large-shape fp64 building blocks (n >= 64): a tiled CTA GEMM on the FP64
// tensor pipe and a blocked triangular solve built on it.
//
// cta_gemm_tiled: C(MxN) = op(A) B with operands in GLOBAL memory (L2 for the
// per-segment scratch), staged through shared memory in BM x 16 / 16 x 64
// tiles by cp.async (double-buffered, zero-filled at the ragged edges); the
// NW warps form an (NW/2) x 2 grid, each warp owning a 16 x 32 block = 2 x 4
// DMMA.8x8x4 fragments, so every k-step issues 8 DMMAs for 6 fragment loads.
#pragma once

#include "plq_device.cuh"

namespace plq {

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// NS = stages of the cp.async ring (2 = double buffering; deeper rings keep
// NS - 1 chunks in flight, which is what hides DRAM latency when the operands'
// L2-resident scratch spills)
template <int NW, int NS = 2>
struct TileCfg {
  static constexpr int BM = 8 * NW, BN = 64, BK = 16;
  static constexpr int LDA = 20, LDB = 68;   // = 4 (mod 8): conflict-free fragment loads
  static constexpr int LDAT = BM + 4;        // transposed A tile (BK x BM), also = 4 (mod 8)
  static_assert(BK * LDAT <= BM * LDA, "transposed A tile fits the A buffer");
  static constexpr int STAGE = BM * LDA + BK * LDB;
  static constexpr int DOUBLES = NS * STAGE;
};

struct NoPre {
  __device__ __forceinline__ double operator()(int, int) const { return 0.0; }
};

// PRE: pre(i, j) (e.g. a Q-block entry in HBM) is loaded before each tile's
// k-loop and the epilogue receives pre(i, j) + acc
// LOWER: tiles that lie entirely above the diagonal (n0 >= m0 + BM) are
// skipped -- for symmetric results whose epilogue writes (i, j <= i) and
// mirrors it.
template <bool TA, int NW, class Epi, bool PRE = false, class Pre = NoPre, int NS = 2, bool LOWER = false>
__device__ __forceinline__ void cta_gemm_tiled(int M, int N, int K, const double* __restrict__ A, int lda,
                                               const double* __restrict__ B, int ldb, double* tiles, Epi epi,
                                               Pre pre = Pre()) {
  using C = TileCfg<NW, NS>;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, LDA = C::LDA, LDB = C::LDB, NT = NW * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  // stage s: A tile at tiles + s * STAGE, B tile behind it
  const int tmc = (M + BM - 1) / BM, tnc = (N + BN - 1) / BN, kc = (K + BK - 1) / BK;
  // 16-byte copies when both operands have even leading dimensions and
  // 16-byte-aligned bases (large-mode scratch); the A tile of a transposed
  // operand is then kept k-major (BK x LDAT) so its pairs stay contiguous
  const bool vec = ((lda | ldb) & 1) == 0 && ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
  for (int tile = 0; tile < tmc * tnc; ++tile) {
    const int m0 = (tile / tnc) * BM, n0 = (tile % tnc) * BN;
    if (LOWER && n0 >= m0 + BM) continue;
    double acc[2][4][2], pv[2][4][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        acc[r][t][0] = acc[r][t][1] = 0.0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = m0 + wr * 16 + r * 8 + g, j = n0 + wc * 32 + t * 8 + 2 * q + e;
          pv[r][t][e] = (PRE && i < M && j < N) ? pre(i, j) : 0.0;
        }
      }
    auto load_vec = [&](int c, int buf) {
      const int k0 = c * BK;
      double* as = tiles + buf * C::STAGE;
      double* bs = as + BM * LDA;
      for (int e = tid; e < BM * BK / 2; e += NT) {
        int i, k;
        if (TA) {
          i = 2 * (e % (BM / 2));
          k = e / (BM / 2);
        } else {
          k = 2 * (e % (BK / 2));
          i = e / (BK / 2);
        }
        const int gi = m0 + i, gk = k0 + k;
        double* dst = TA ? as + k * C::LDAT + i : as + i * LDA + k;
        if (TA) {
          const double* src = A + (size_t)gk * lda + gi;
          if (gk < K && gi + 1 < M) {
            cp_async16(dst, src);
          } else {
            cp_async8(dst, gk < K && gi < M ? src : A, gk < K && gi < M);
            cp_async8(dst + 1, gk < K && gi + 1 < M ? src + 1 : A, gk < K && gi + 1 < M);
          }
        } else {
          const double* src = A + (size_t)gi * lda + gk;
          if (gi < M && gk + 1 < K) {
            cp_async16(dst, src);
          } else {
            cp_async8(dst, gi < M && gk < K ? src : A, gi < M && gk < K);
            cp_async8(dst + 1, gi < M && gk + 1 < K ? src + 1 : A, gi < M && gk + 1 < K);
          }
        }
      }
      for (int e = tid; e < BK * BN / 2; e += NT) {
        const int k = e / (BN / 2), j = 2 * (e % (BN / 2));
        const int gk = k0 + k, gj = n0 + j;
        const double* src = B + (size_t)gk * ldb + gj;
        double* dst = bs + k * LDB + j;
        if (gk < K && gj + 1 < N) {
          cp_async16(dst, src);
        } else {
          cp_async8(dst, gk < K && gj < N ? src : B, gk < K && gj < N);
          cp_async8(dst + 1, gk < K && gj + 1 < N ? src + 1 : B, gk < K && gj + 1 < N);
        }
      }
    };
    auto load = [&](int c, int buf) {
      if (vec) {
        load_vec(c, buf);
        return;
      }
      const int k0 = c * BK;
      double* as = tiles + buf * C::STAGE;
      double* bs = as + BM * LDA;
      for (int e = tid; e < BM * BK; e += NT) {
        int i, k;
        if (TA) {
          i = e % BM;
          k = e / BM;
        } else {
          k = e % BK;
          i = e / BK;
        }
        const int gi = m0 + i, gk = k0 + k;
        const bool v = gi < M && gk < K;
        const double* src = v ? (TA ? A + (size_t)gk * lda + gi : A + (size_t)gi * lda + gk) : A;
        cp_async8(as + i * LDA + k, src, v);
      }
      for (int e = tid; e < BK * BN; e += NT) {
        const int k = e / BN, j = e % BN;
        const int gk = k0 + k, gj = n0 + j;
        const bool v = gk < K && gj < N;
        cp_async8(bs + k * LDB + j, v ? B + (size_t)gk * ldb + gj : B, v);
      }
    };
    // ring of NS stages: chunks c .. c + NS - 2 in flight while chunk c is
    // consumed; one commit group per chunk slot (empty past the end), so
    // wait_group<NS - 2> always means "chunk c has landed"
#pragma unroll
    for (int st = 0; st < NS - 1; ++st) {
      if (st < kc) load(st, st);
      cp_async_commit();
    }
    for (int c = 0; c < kc; ++c) {
      cp_async_wait<NS - 2>();
      __syncthreads();   // chunk c visible to all; everyone is done with chunk c - 1's buffer
      if (c + NS - 1 < kc) load(c + NS - 1, (c + NS - 1) % NS);
      cp_async_commit();
      const double* as = tiles + (c % NS) * C::STAGE;
      const double* bs = as + BM * LDA;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[2], bf[4];
#pragma unroll
        for (int r = 0; r < 2; ++r)
          af[r] = (TA && vec) ? as[(kk + q) * C::LDAT + wr * 16 + r * 8 + g] : as[(wr * 16 + r * 8 + g) * LDA + kk + q];
#pragma unroll
        for (int t = 0; t < 4; ++t) bf[t] = bs[(kk + q) * LDB + wc * 32 + t * 8 + g];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < 4; ++t) dmma884(acc[r][t][0], acc[r][t][1], af[r], bf[t]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();   // the next tile's prologue reuses the buffers
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = m0 + wr * 16 + r * 8 + g, j = n0 + wc * 32 + t * 8 + 2 * q + e;
          if (i < M && j < N) epi(i, j, PRE ? pv[r][t][e] + acc[r][t][e] : acc[r][t][e]);
        }
  }
}

// X <- (L L')^{-1} X for the m x W block X (cho_solve), blocked by 8 rows:
// the off-diagonal updates are DMMA GEMMs over all W columns, the 8 x 8
// diagonal solves go thread per column.  `L` and `X` may be global or shared.
__device__ __forceinline__ void cta_cho_solve_blocked(const double* L, int m, int ldl, double* X, int W, int ldx) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // forward: L y = x
  for (int r0 = 0; r0 < m; r0 += 8) {
    const int rb = min(8, m - r0);
    if (r0 > 0) {
      cta_gemm<false, false, 1, 1>(rb, W, r0, L + (size_t)r0 * ldl, ldl, X, ldx,
                                   [&](int i, int j, double acc) { X[(size_t)(r0 + i) * ldx + j] -= acc; });
      __syncthreads();
    }
    for (int c = tid; c < W; c += nt) {
      double y[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < rb) {
          double v = X[(size_t)(r0 + i) * ldx + c];
#pragma unroll
          for (int k = 0; k < i; ++k) v -= L[(size_t)(r0 + i) * ldl + r0 + k] * y[k];
          y[i] = v / L[(size_t)(r0 + i) * ldl + r0 + i];
          X[(size_t)(r0 + i) * ldx + c] = y[i];
        }
      }
    }
    __syncthreads();
  }
  // backward: L' x = y
  const int nb = (m + 7) / 8;
  for (int bb = nb - 1; bb >= 0; --bb) {
    const int r0 = bb * 8, rb = min(8, m - r0), r1 = r0 + rb;
    if (r1 < m) {
      // X[r0:r1] -= (L')[r0:r1, r1:m] X[r1:m] ; (L')(i,k) = L[r1+k][r0+i]
      cta_gemm<true, false, 1, 1>(rb, W, m - r1, L + (size_t)r1 * ldl + r0, ldl, X + (size_t)r1 * ldx, ldx,
                                  [&](int i, int j, double acc) { X[(size_t)(r0 + i) * ldx + j] -= acc; });
      __syncthreads();
    }
    for (int c = tid; c < W; c += nt) {
      double y[8];
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        if (i < rb) {
          double v = X[(size_t)(r0 + i) * ldx + c];
#pragma unroll
          for (int k = i + 1; k < 8; ++k)
            if (k < rb) v -= L[(size_t)(r0 + k) * ldl + r0 + i] * y[k];
          y[i] = v / L[(size_t)(r0 + i) * ldl + r0 + i];
          X[(size_t)(r0 + i) * ldx + c] = y[i];
        }
      }
    }
    __syncthreads();
  }
}

// forward substitution only: X <- L^{-1} X, blocked
__device__ __forceinline__ void cta_trsm_lower_blocked(const double* L, int m, int ldl, double* X, int W, int ldx) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int r0 = 0; r0 < m; r0 += 8) {
    const int rb = min(8, m - r0);
    if (r0 > 0) {
      cta_gemm<false, false, 1, 1>(rb, W, r0, L + (size_t)r0 * ldl, ldl, X, ldx,
                                   [&](int i, int j, double acc) { X[(size_t)(r0 + i) * ldx + j] -= acc; });
      __syncthreads();
    }
    for (int c = tid; c < W; c += nt) {
      double y[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < rb) {
          double v = X[(size_t)(r0 + i) * ldx + c];
#pragma unroll
          for (int k = 0; k < i; ++k) v -= L[(size_t)(r0 + i) * ldl + r0 + k] * y[k];
          y[i] = v / L[(size_t)(r0 + i) * ldl + r0 + i];
          X[(size_t)(r0 + i) * ldx + c] = y[i];
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace plq
