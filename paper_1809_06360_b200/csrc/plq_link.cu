// K2: the link-point coupling solve.
//
// The reference assembles the multiplier-matching equations over the J-1
// interior links (parallel.py:286-319) and solves the SPD block-tridiagonal
// system (-diag, -sub) x = rhs by sequential block Cholesky
// (LinkSystem.solve parallel.py:264-283 -> endpoint.solve_block_tridiagonal
// endpoint.py:410-438).  A J-1 = 1023-deep sequential chain is the GPU's
// sequential-depth risk, so here it is solved by block cyclic reduction:
// each level eliminates the odd blocks in parallel (one CTA each), leaving a
// half-size SPD block-tridiagonal system on the even blocks; log2(J) levels
// down, back-substitution climbs up again.  Per eliminated block i with
// Cholesky D_i = L L' and W = L^{-1} [A(i,i-1) | A(i,i+1) | b_i]:
//   D_{i-1} -= W_L'W_L,  D_{i+1} -= W_R'W_R,  A'(i+1,i-1) = -W_R'W_L,
//   b_{i-1} -= W_L'W_b,  b_{i+1} -= W_R'W_b,  x_i = L^{-T}(W_b - W_L x_{i-1} - W_R x_{i+1}).
// A pivot block that is not positive-definite raises LinkSingular, as the
// reference does (parallel.py:267-271).
#include "plq_device.cuh"
#include "plq_blocked.cuh"
#include "plq_gemm.cuh"
#include "plq_internal.h"
#include "plq_tma.cuh"

#include <cstdlib>
#include <vector>

namespace plq {

namespace {

struct LinkLevel {
  double* D;     // (B,K,n,n)   SPD diagonal blocks
  double* S;     // (B,K-1,n,n) S[i] = A(i+1,i)
  double* rhs;   // (B,K,n)
  double* x;     // (B,K,n)     solution of this level's system
  double* Lc;    // (B,E,n,n)   Cholesky factors of eliminated blocks
  double* Wm;    // (B,E,n,2n+1)
  double* CL;    // (B,E,n,n)
  double* CR;    // (B,E,n,n)
  double* X;     // (B,E,n,n)
  double* cL;    // (B,E,n)
  double* cR;    // (B,E,n)
  double* Linv;  // (B,E,ceil(n/8)*64) diagonal-block inverses (split path)
  int K, E, top;
};

struct LinkPlan {
  std::vector<LinkLevel> lv;
  double* rpart;   // (B, K0) link-residual partials
  size_t doubles;
};

LinkPlan plan_link(int64_t B, int J, int n, double* base) {
  LinkPlan P;
  P.rpart = nullptr;
  P.doubles = 0;
  if (J < 2) return P;   // a single segment has no links
  const int64_t nn = (int64_t)n * n, w = 2 * n + 1;
  size_t off = 0;
  auto take = [&](int64_t count) {
    double* p = base ? base + off : nullptr;
    off += (size_t)((count + 1) & ~1LL);
    return p;
  };
  int K = J - 1;
  while (true) {
    LinkLevel L{};
    L.K = K;
    L.top = (K == 1);
    L.E = L.top ? 1 : K / 2;
    L.D = take(B * K * nn);
    L.S = take(B * (K > 1 ? K - 1 : 0) * nn);
    L.rhs = take(B * K * n);
    L.x = take(B * K * n);
    L.Lc = take(B * L.E * nn);
    L.Wm = take(B * L.E * n * w);
    L.CL = take(B * L.E * nn);
    L.CR = take(B * L.E * nn);
    L.X = take(B * L.E * nn);
    L.cL = take(B * L.E * n);
    L.cR = take(B * L.E * n);
    L.Linv = take(B * L.E * ((n + 7) / 8) * 64);
    P.lv.push_back(L);
    if (L.top) break;
    K = (K + 1) / 2;
  }
  P.rpart = take(B * (J - 1));
  P.doubles = off;
  return P;
}


// Stage contiguous global blocks into shared memory with one bulk copy each
// (one memory latency for the whole set instead of one per loop trip).
// Falls back to a plain cooperative copy when a block is not a multiple of
// 16 bytes or not 16-byte aligned (odd n).
struct BulkSet {
  static constexpr int MAXB = 6;
  double* dst[MAXB];
  const double* src[MAXB];
  int count[MAXB];
  int nb = 0;
  __device__ void add(double* d, const double* s, int c) {
    dst[nb] = d;
    src[nb] = s;
    count[nb] = c;
    ++nb;
  }
};

__device__ __forceinline__ void bulk_stage(BulkSet& bs, uint64_t* bar, uint32_t& phase) {
  bool ok = true;
  for (int k = 0; k < bs.nb; ++k)
    ok = ok && ((bs.count[k] * 8) % 16 == 0) && ((reinterpret_cast<uintptr_t>(bs.src[k]) & 15) == 0) &&
         ((reinterpret_cast<uintptr_t>(bs.dst[k]) & 15) == 0);
  if (ok) {
    if (threadIdx.x == 0) {
      uint32_t bytes = 0;
      for (int k = 0; k < bs.nb; ++k) bytes += 8u * bs.count[k];
      fence_proxy_async();
      mbar_arrive_tx(bar, bytes);
      for (int k = 0; k < bs.nb; ++k) bulk_g2s(bs.dst[k], bs.src[k], 8u * bs.count[k], bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
  } else {
    for (int k = 0; k < bs.nb; ++k)
      for (int i = threadIdx.x; i < bs.count[k]; i += blockDim.x) bs.dst[k][i] = bs.src[k][i];
  }
  __syncthreads();
}

// level-0 system from the segment-start value blocks (parallel.py:286-319):
// D_i = Vzz0_i + Vxx0_{i+1},  A(i+1,i) = Vzx0_{i+1},
// b_i = -vz1_i - vx1_{i+1} (- Vzx0_0 x_init for i = 0).
__global__ void link_assemble0(plq_problem_t p, const double* vf0, LinkLevel L, double* link_residual) {
  const int n = p.n, J = p.J, K = L.K;
  const int64_t nn = (int64_t)n * n, vsz = 3 * nn + 2 * n;
  const int64_t b = blockIdx.x / K;
  const int i = blockIdx.x % K;
  if (i == 0 && threadIdx.x == 0) link_residual[b] = 0.0;   // link_residual_part accumulates the maximum
  const double* left = vf0 + (b * J + i) * vsz;
  const double* right = vf0 + (b * J + i + 1) * vsz;
  double* D = L.D + (b * K + i) * nn;
  for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) D[idx] = left[2 * nn + idx] + right[idx];
  if (i + 1 < K) {
    double* S = L.S + (b * (K - 1) + i) * nn;
    const double* rr = vf0 + (b * J + i + 1) * vsz;   // segment i+1 is an endpoint segment here
    for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) S[idx] = rr[nn + idx];
  }
  double* rhs = L.rhs + (b * K + i) * n;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double v = -left[3 * nn + n + r] + -right[3 * nn + r];
    if (i == 0) {
      double s = 0.0;
      for (int c = 0; c < n; ++c) s += left[nn + r * n + c] * p.x_init[b * n + c];
      v += -s;
    }
    rhs[r] = v;
  }
}

__device__ __forceinline__ void flag_singular(plq_problem_t& p, int32_t* status, int64_t b) {
  if (threadIdx.x == 0 && status[b * p.J] == 0) status[b * p.J] = PLQ_STATUS_LINK_SINGULAR;
}

// offset (doubles) of the blocked-factorization scratch in link_eliminate's
// dynamic shared memory: after the factor / right-hand sides / staging (n <=
// 64) or the factor / GEMM tiles (n > 64); 2 * ceil(n/8) * 64 + 8 * 64 doubles
__host__ __device__ inline size_t link_elim_blocked_off(int n, bool sm, bool lsm, int ldl, int ldw, int threads) {
  if (sm) return ((((size_t)n * ldl + (size_t)n * ldw + 1) & ~size_t(1)) + 3 * (size_t)n * n + n + 1) & ~size_t(1);
  return (lsm ? (((size_t)n * ldl + 1) & ~size_t(1)) : 0) + (threads == 256 ? (size_t)TileCfg<8>::DOUBLES : 0);
}
__host__ __device__ inline size_t link_elim_blocked_doubles(int n) { return 2 * (size_t)((n + 7) / 8) * 64 + 8 * 64; }

// eliminate the odd blocks of one level (or the single top block).  For
// n <= 64 the pivot block and W live in shared memory; the factor and W are
// written back to global once for the back-substitution.
//
// FUSED (levels >= 1, n <= 64): the level's system is not assembled by a
// separate launch.  The grid has one CTA per block of the level: CTA k builds
// block k from the previous level's even block 2k and its eliminated
// neighbours' Schur terms (D = D'_{2k} - CR'_{k-1} - CL'_k, A(k+1,k) = -X'_k,
// rhs likewise) -- kept (even) blocks are written out for the next level and
// the CTA exits, odd blocks (and the top block) are assembled straight into
// the factor / W buffers and eliminated.  One launch and one ~12 us
// dependent-latency step less per level; the S blocks of levels >= 1 are
// never materialized (only odd blocks read them).
// MINB: resident CTAs per SM the register allocation is bounded for -- 2 (128
// registers) for the wide levels, 1 (no cap) for levels with at most one CTA
// per SM anyway.
template <bool FUSED, int MINB>
__global__ void __launch_bounds__(256, MINB)
    link_eliminate(plq_problem_t p, LinkLevel L, LinkLevel Pv, int32_t* status, int fused_solve) {
  __shared__ int flag;
  extern __shared__ __align__(16) double dsm[];
  const int n = p.n, K = L.K, E = L.E, w = 2 * n + 1;
  const int64_t nn = (int64_t)n * n;
  const int per = FUSED ? K : E;
  const int64_t b = blockIdx.x / per;
  const int kb = blockIdx.x % per;
  const int o = FUSED ? kb / 2 : kb;
  const int i = L.top ? 0 : (FUSED ? kb : 2 * o + 1);
  // previous level's pieces of block i (FUSED)
  const int Kp = Pv.K, Ep = Pv.E;
  const bool pl = FUSED && i >= 1, pr = FUSED && 2 * i + 1 < Kp;
  const double* pD = FUSED ? Pv.D + (b * Kp + 2 * i) * nn : nullptr;
  const double* pCR = pl ? Pv.CR + (b * Ep + (i - 1)) * nn : nullptr;
  const double* pCL = pr ? Pv.CL + (b * Ep + i) * nn : nullptr;
  const double* prh = FUSED ? Pv.rhs + (b * Kp + 2 * i) * n : nullptr;
  const double* pcR = pl ? Pv.cR + (b * Ep + (i - 1)) * n : nullptr;
  const double* pcL = pr ? Pv.cL + (b * Ep + i) * n : nullptr;
  if (FUSED && !L.top && (kb & 1) == 0) {
    // kept block: next level's input
    double* Dn = L.D + (b * K + i) * nn;
    for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) {
      double v = pD[idx];
      if (pl) v -= pCR[idx];
      if (pr) v -= pCL[idx];
      Dn[idx] = v;
    }
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double v = prh[r];
      if (pl) v -= pcR[r];
      if (pr) v -= pcL[r];
      L.rhs[(b * K + i) * n + r] = v;
    }
    return;
  }
  const bool sm = n <= 64;     // factor and right-hand sides on chip
  const bool lsm = n <= 128;   // the factor on chip (n <= 128: 132 KB), W in L2
  const int ldl = lsm ? n + 1 : n;
  const int ldw = sm ? ((w + 3) / 8) * 8 + 4 : w;
  double* gLc = L.Lc + (b * E + o) * nn;
  double* gWm = L.Wm + (b * E + o) * n * w;
  double* Lc = lsm ? dsm : gLc;
  double* Wm = sm ? dsm + n * ldl : gWm;
  double* tiles = sm ? nullptr : dsm + (lsm ? ((n * ldl + 1) & ~1) : 0);
  const double* D = FUSED ? pD : L.D + (b * K + i) * nn;
  const bool has_l = i >= 1, has_r = i + 1 < K;
  // A(i,i-1) and A(i+1,i) (A(i,i+1) = Sr'); FUSED: minus the previous level's X blocks
  const double* Sl = has_l ? (FUSED ? Pv.X + (b * Ep + (i - 1)) * nn : L.S + (b * (K - 1) + (i - 1)) * nn) : nullptr;
  const double* Sr = has_r ? (FUSED ? Pv.X + (b * Ep + i) * nn : L.S + (b * (K - 1) + i) * nn) : nullptr;
  const double* rh = FUSED ? prh : L.rhs + (b * K + i) * n;
  const double ssign = FUSED ? -1.0 : 1.0;
  if (sm) {
    // bulk-stage D, S_l, S_r, rhs behind the factor / W buffers, assemble in smem
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    double* st = dsm + ((n * ldl + n * ldw + 1) & ~1);
    BulkSet bs;
    bs.add(st, D, (int)nn);
    if (has_l) bs.add(st + nn, Sl, (int)nn);
    if (has_r) bs.add(st + 2 * nn, Sr, (int)nn);
    bs.add(st + 3 * nn, rh, n);
    bulk_stage(bs, &bar, phase);
    for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) {
      double v = st[idx];
      if (pl) v -= pCR[idx];
      if (pr) v -= pCL[idx];
      Lc[(idx / n) * ldl + idx % n] = v;
    }
    for (int idx = threadIdx.x; idx < n * w; idx += blockDim.x) {
      const int r = idx / w, c = idx % w;
      double v;
      if (c < n)
        v = has_l ? ssign * st[nn + r * n + c] : 0.0;
      else if (c < 2 * n)
        v = has_r ? ssign * st[2 * nn + (c - n) * n + r] : 0.0;
      else {
        v = st[3 * nn + r];
        if (pl) v -= pcR[r];
        if (pr) v -= pcL[r];
      }
      Wm[r * ldw + c] = v;
    }
  } else {
    for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) Lc[(idx / n) * ldl + idx % n] = D[idx];
    for (int idx = threadIdx.x; idx < n * w; idx += blockDim.x) {
      const int r = idx / w, c = idx % w;
      double v;
      if (c < n)
        v = has_l ? Sl[r * n + c] : 0.0;
      else if (c < 2 * n)
        v = has_r ? Sr[(c - n) * n + r] : 0.0;
      else
        v = rh[r];
      Wm[r * ldw + c] = v;
    }
  }
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  // blocked Cholesky / forward solve (plq_blocked.cuh) for 8-warp CTAs; the
  // scratch (block inverses, diagonal staging, warp tiles) follows the layout
  const bool blocked = n >= 16 && blockDim.x == 256;
  double* bsc = dsm + link_elim_blocked_off(n, sm, lsm, ldl, ldw, blockDim.x);
  auto csync = [] { __syncthreads(); };
  const int nbk = (n + 7) / 8;
  // W on chip: the forward solve W <- L^{-1} W rides in the factorization's
  // trailing phases (block row k of W next to step k's Schur tiles: n/8
  // group barriers less than a separate gtrsm8)
  const bool fsolve = blocked && sm && fused_solve;
  const bool ok = blocked ? gchol8<8>(Lc, n, ldl, bsc, &flag, threadIdx.x, csync, bsc + nbk * 64,
                                      fsolve ? Wm : nullptr, w, ldw, bsc + 2 * nbk * 64)
                          : cta_cholesky(Lc, n, ldl, &flag);
  if (!ok) {
    flag_singular(p, status, b);
    return;
  }
  if (fsolve) {
  } else if (blocked)
    gtrsm8<0, 8>(Lc, n, ldl, bsc, Wm, w, ldw, bsc + 2 * nbk * 64, threadIdx.x, csync);
  else if (n >= 16)
    cta_trsm_lower_blocked(Lc, n, ldl, Wm, w, ldw);
  else
    cta_trsm_lower(Lc, n, ldl, Wm, w, ldw);
  if (lsm)
    for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) gLc[idx] = Lc[(idx / n) * ldl + idx % n];
  if (sm)
    for (int idx = threadIdx.x; idx < n * w; idx += blockDim.x) gWm[idx] = Wm[(idx / w) * ldw + idx % w];
  if (L.top) {
    // top block: nothing left to couple to -- finish x = L^{-T} W_b here
    // (n <= 64: the factor and W are on chip), no back-substitution launch
    if (sm) {
      double* v = dsm + ((n * ldl + n * ldw + 1) & ~1);   // staging area, dead
      __syncthreads();
      for (int r = threadIdx.x; r < n; r += blockDim.x) v[r] = Wm[r * ldw + 2 * n];
      __syncthreads();
      for (int r = n - 1; r >= 0; --r) {
        if (threadIdx.x == 0) v[r] /= Lc[r * ldl + r];
        __syncthreads();
        const double xr_ = v[r];
        for (int k = threadIdx.x; k < r; k += blockDim.x) v[k] -= Lc[r * ldl + k] * xr_;
        __syncthreads();
      }
      for (int r = threadIdx.x; r < n; r += blockDim.x) L.x[b * K * n + r] = v[r];
    }
    return;
  }
  double* CL = L.CL + (b * E + o) * nn;
  double* CR = L.CR + (b * E + o) * nn;
  double* X = L.X + (b * E + o) * nn;
  double* cL = L.cL + (b * E + o) * n;
  double* cR = L.cR + (b * E + o) * n;
  auto gram = [&](int r, int c, double acc) {
    if (r < n) {
      if (c < n)
        CL[r * n + c] = acc;
      else if (c == 2 * n)
        cL[r] = acc;
    } else {
      const int rr = r - n;
      if (c < n)
        X[rr * n + c] = acc;
      else if (c < 2 * n)
        CR[rr * n + (c - n)] = acc;
      else
        cR[rr] = acc;
    }
  };
  if (!sm && blockDim.x == 256)
    cta_gemm_tiled<true, 8>(2 * n, w, n, Wm, w, Wm, w, tiles, gram);
  else
    cta_gemm<true, false, 2, 2>(2 * n, w, n, Wm, ldw, Wm, ldw, gram);   // 16 x 16 per warp: half the fragment loads per DMMA
}

// ---- large blocks (n > 64): one elimination split over many CTAs ---------
// The elimination of a level is its critical path, and the deep levels have
// only a few blocks (cfg3: 127, 64, ..., 1 of n = 128), so for n > 64 each
// block's elimination runs as three kernels: the blocked Cholesky (one CTA
// per block), the forward solve W = L^{-1}[A(i,i-1) | A(i,i+1) | b_i] in
// column slabs (link_slabs() CTAs per block), and the Gram products in 64 x 64
// tiles (LINK_GRAM_TILES CTAs per block).  Same arithmetic as link_eliminate.
constexpr int LINK_SLAB_LD = 76;     // widest slab: ceil(w/32)*8 <= 72 for n <= 128, stride = 4 (mod 8)

// Column slabs of W (w = 2n+1 columns) per eliminated block: four CTAs while
// the level has enough blocks to fill the GPU, eight at the deep levels (few
// blocks: the slab solve is a latency chain of n/8 block steps whose length
// per step is the number of 8-column tiles a warp owns)
__host__ __device__ inline int link_slabs(int64_t blocks) { return blocks * 4 <= 74 ? 8 : 4; }

__host__ __device__ inline int link_ldl_big(int n) { return n + ((12 - n % 8) % 8); }   // = 4 (mod 8)

__host__ __device__ inline void link_slab(int w, int sidx, int slabs, int* c0, int* c1) {
  const int base = ((w + 8 * slabs - 1) / (8 * slabs)) * 8;   // multiple of 8 (72 x 3 + 41 or 40 x 6 + 17 at n = 128)
  *c0 = min(w, sidx * base);
  *c1 = (sidx == slabs - 1) ? w : min(w, (sidx + 1) * base);
}

// Stage an n x n row-major global block into shared memory with row stride
// ld (= 4 mod 8, rows 16-byte aligned) by one bulk copy per row (TMA 1-D),
// plus an optional contiguous extra range; falls back to a cooperative copy
// when a row is not a multiple of 16 bytes.
__device__ __forceinline__ void stage_rows(double* dst, int ld, const double* src, int n, double* xdst,
                                           const double* xsrc, int xcount, uint64_t* bar, uint32_t& phase) {
  if ((n % 2) == 0 && (ld % 2) == 0 && (xcount % 2) == 0) {
    if (threadIdx.x < 32) {   // row copies spread over warp 0's lanes (one issuer serializes them)
      const int lane = threadIdx.x;
      fence_proxy_async();
      if (lane == 0) mbar_arrive_tx(bar, 8u * (uint32_t)(n * n + xcount));
      __syncwarp();
      for (int r = lane; r < n; r += 32) bulk_g2s(dst + (size_t)r * ld, src + (size_t)r * n, 8u * n, bar);
      if (xcount && lane == 0) bulk_g2s(xdst, xsrc, 8u * xcount, bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
  } else {
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) dst[(idx / n) * ld + idx % n] = src[idx];
    for (int idx = threadIdx.x; idx < xcount; idx += blockDim.x) xdst[idx] = xsrc[idx];
  }
  __syncthreads();
}

// (16 warps: the trailing update of a 128 x 128 block has up to 120 tiles per block step)
__global__ void __launch_bounds__(512) link_factor_big(plq_problem_t p, LinkLevel L, int32_t* status) {
  __shared__ int flag;
  extern __shared__ __align__(16) double dsm[];
  __shared__ __align__(8) uint64_t bar;
  const int n = p.n, K = L.K, E = L.E, ldl = link_ldl_big(n), nbk = (n + 7) / 8;
  const int64_t nn = (int64_t)n * n;
  const int64_t b = blockIdx.x / E;
  const int o = blockIdx.x % E;
  const int i = L.top ? 0 : 2 * o + 1;
  const double* D = L.D + (b * K + i) * nn;
  double* Lc = dsm;
  double* Ld = dsm + (((size_t)n * ldl + 1) & ~size_t(1));
  double* Linv = L.Linv + (b * E + o) * nbk * 64;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    flag = 0;
  }
  __syncthreads();
  uint32_t phase = 0;
  stage_rows(Lc, ldl, D, n, nullptr, nullptr, 0, &bar, phase);
  if (!gchol8<16>(Lc, n, ldl, Linv, &flag, threadIdx.x, [] { __syncthreads(); }, Ld)) {
    flag_singular(p, status, b);
    return;
  }
  double* gLc = L.Lc + (b * E + o) * nn;
  for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) {
    const int r = idx / n, c = idx % n;
    gLc[idx] = c <= r ? Lc[r * ldl + c] : 0.0;
  }
}

__global__ void __launch_bounds__(256) link_trsm_big(plq_problem_t p, LinkLevel L, const int32_t* status) {
  extern __shared__ __align__(16) double dsm[];
  const int n = p.n, K = L.K, E = L.E, w = 2 * n + 1, nbk = (n + 7) / 8;
  const int64_t nn = (int64_t)n * n;
  const int slabs = link_slabs((int64_t)p.B * E);
  const int64_t b = blockIdx.x / (E * slabs);
  const int o = (blockIdx.x / slabs) % E;
  const int sidx = blockIdx.x % slabs;
  if (status[b * p.J] == PLQ_STATUS_LINK_SINGULAR) return;
  const int i = L.top ? 0 : 2 * o + 1;
  int c0, c1;
  link_slab(w, sidx, slabs, &c0, &c1);
  const int sw = c1 - c0;
  const bool has_l = !L.top && i >= 1, has_r = !L.top && i + 1 < K;
  const double* Sl = has_l ? L.S + (b * (K - 1) + (i - 1)) * nn : nullptr;
  const double* Sr = has_r ? L.S + (b * (K - 1) + i) * nn : nullptr;
  const double* rh = L.rhs + (b * K + i) * n;
  const double* gLc = L.Lc + (b * E + o) * nn;
  const int lls = link_ldl_big(n);
  double* Ls = dsm;                                   // n x lls (factor)
  double* Li = Ls + (size_t)n * lls;                  // nbk * 64
  double* X = Li + nbk * 64;                          // n x LINK_SLAB_LD
  double* wsc = X + (size_t)n * LINK_SLAB_LD;          // 8 * 64
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  // factor rows and the block inverses by bulk copies, overlapping the slab assembly
  if ((n % 2) == 0 && threadIdx.x < 32) {   // row copies over warp 0's lanes
    const int lane = threadIdx.x;
    fence_proxy_async();
    if (lane == 0) mbar_arrive_tx(&bar, 8u * (uint32_t)(nn + nbk * 64));
    __syncwarp();
    for (int r = lane; r < n; r += 32) bulk_g2s(Ls + (size_t)r * lls, gLc + (size_t)r * n, 8u * n, &bar);
    if (lane == 0) bulk_g2s(Li, L.Linv + (b * E + o) * nbk * 64, 8u * nbk * 64, &bar);
  }
  if ((n % 2) != 0) {
    for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) Ls[(idx / n) * lls + idx % n] = gLc[idx];
    for (int idx = threadIdx.x; idx < nbk * 64; idx += blockDim.x) Li[idx] = L.Linv[(b * E + o) * nbk * 64 + idx];
  }
  for (int idx = threadIdx.x; idx < n * sw; idx += blockDim.x) {
    const int r = idx / sw, c = c0 + idx % sw;
    double v;
    if (c < n)
      v = has_l ? Sl[r * n + c] : 0.0;
    else if (c < 2 * n)
      v = has_r ? Sr[(c - n) * n + r] : 0.0;
    else
      v = rh[r];
    X[r * LINK_SLAB_LD + (c - c0)] = v;
  }
  if ((n % 2) == 0) mbar_wait(&bar, phase);
  __syncthreads();
  gtrsm8<0, 8>(Ls, n, lls, Li, X, sw, LINK_SLAB_LD, wsc, threadIdx.x, [] { __syncthreads(); });
  double* gWm = L.Wm + (b * E + o) * n * w;
  for (int idx = threadIdx.x; idx < n * sw; idx += blockDim.x) {
    const int r = idx / sw, c = idx % sw;
    gWm[r * w + c0 + c] = X[r * LINK_SLAB_LD + c];
  }
}

// Gram tiles of W'W: CL = W_L'W_L, X = W_R'W_L, CR = W_R'W_R (n x n each, in
// 64 x 64 tiles), cL = W_L'W_b, cR = W_R'W_b (one 2n x 1 column, tile 0 of
// the extra row).  grid = B * E * (3 * (n/64)^2 + 1)
__global__ void __launch_bounds__(256) link_gram_big(plq_problem_t p, LinkLevel L, const int32_t* status) {
  extern __shared__ __align__(16) double tiles[];
  const int n = p.n, E = L.E, w = 2 * n + 1, nt = (n + 63) / 64, per = 3 * nt * nt + 1;
  const int64_t nn = (int64_t)n * n;
  const int64_t b = blockIdx.x / (E * per);
  const int o = (blockIdx.x / per) % E;
  const int t = blockIdx.x % per;
  if (status[b * p.J] == PLQ_STATUS_LINK_SINGULAR) return;
  const double* Wm = L.Wm + (b * E + o) * n * w;
  double* CL = L.CL + (b * E + o) * nn;
  double* CR = L.CR + (b * E + o) * nn;
  double* Xo = L.X + (b * E + o) * nn;
  if (t == per - 1) {
    // [cL; cR] = [W_L W_R]' W_b : 2n outputs, thread per output
    for (int r = threadIdx.x; r < 2 * n; r += blockDim.x) {
      double acc = 0.0;
#pragma unroll 8
      for (int k = 0; k < n; ++k) acc += Wm[k * w + r] * Wm[k * w + 2 * n];
      if (r < n)
        L.cL[(b * E + o) * n + r] = acc;
      else
        L.cR[(b * E + o) * n + r - n] = acc;
    }
    return;
  }
  const int blk = t / (nt * nt), tt = t % (nt * nt), ti = tt / nt, tj = tt % nt;
  // blk 0: CL (rows W_L, cols W_L); 1: X (rows W_R, cols W_L); 2: CR (rows W_R, cols W_R)
  const int ra = (blk == 0 ? 0 : n) + ti * 64, cb = (blk == 2 ? n : 0) + tj * 64;
  double* dst = blk == 0 ? CL : (blk == 1 ? Xo : CR);
  const int M = min(64, n - ti * 64), N = min(64, n - tj * 64);
  cta_gemm_tiled<true, 8>(M, N, n, Wm + ra, w, Wm + cb, w, tiles,
                          [&](int r, int c, double acc) { dst[(ti * 64 + r) * n + tj * 64 + c] = acc; });
}

// next level's system on the even blocks
__global__ void link_assemble_next(plq_problem_t p, LinkLevel L, LinkLevel N) {
  const int n = p.n, K = L.K, E = L.E, K2 = N.K;
  const int64_t nn = (int64_t)n * n;
  const int64_t b = blockIdx.x / K2;
  const int e2 = blockIdx.x % K2;
  const int e = 2 * e2;
  const bool has_l = e >= 2, has_r = e + 1 < K;
  const double* D = L.D + (b * K + e) * nn;
  double* Dn = N.D + (b * K2 + e2) * nn;
  const double* CRl = has_l ? L.CR + (b * E + (e2 - 1)) * nn : nullptr;
  const double* CLr = has_r ? L.CL + (b * E + e2) * nn : nullptr;
  for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) {
    double v = D[idx];
    if (has_l) v -= CRl[idx];
    if (has_r) v -= CLr[idx];
    Dn[idx] = v;
  }
  if (e2 >= 1) {
    const double* X = L.X + (b * E + (e2 - 1)) * nn;
    double* Sn = N.S + (b * (K2 - 1) + (e2 - 1)) * nn;
    for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) Sn[idx] = -X[idx];
  }
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double v = L.rhs[(b * K + e) * n + r];
    if (has_l) v -= L.cR[(b * E + (e2 - 1)) * n + r];
    if (has_r) v -= L.cL[(b * E + e2) * n + r];
    N.rhs[(b * K2 + e2) * n + r] = v;
  }
}

// back-substitution of one level: x_i = L^{-T} (W_b - W_L x_{i-1} - W_R x_{i+1})
// for eliminated blocks, copy from the coarser level for kept blocks.
__global__ void link_backsub(plq_problem_t p, LinkLevel L, LinkLevel C, int has_coarse) {
  extern __shared__ __align__(16) double v[];
  const int n = p.n, K = L.K, E = L.E, w = 2 * n + 1;
  const int64_t nn = (int64_t)n * n;
  const int64_t b = blockIdx.x / K;
  const int i = blockIdx.x % K;
  double* x = L.x + (b * K + i) * n;
  const bool elim = L.top ? true : (i & 1);
  if (!elim) {
    for (int r = threadIdx.x; r < n; r += blockDim.x) x[r] = C.x[(b * C.K + i / 2) * n + r];
    return;
  }
  const int o = L.top ? 0 : (i - 1) / 2;
  const double* Lc = L.Lc + (b * E + o) * nn;
  const double* Wm = L.Wm + (b * E + o) * n * w;
  const bool has_l = !L.top && i >= 1, has_r = !L.top && i + 1 < K;
  const double* xl = has_l ? C.x + (b * C.K + (i - 1) / 2) * n : nullptr;
  const double* xr = has_r ? C.x + (b * C.K + (i + 1) / 2) * n : nullptr;
  (void)has_coarse;
  const bool sm = n <= 64;
  double* Ls = v + n + 2;   // n x (n+1) when staged
  const int ldl = n + 1;
  if (sm) {
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    double* st = Ls + ((n * ldl + 1) & ~1);        // raw L (nn), W (n*w), xl, xr
    BulkSet bs;
    bs.add(st, Lc, (int)nn);
    bs.add(st + nn, Wm, n * w);
    if (has_l) bs.add(st + nn + n * w + (n * w & 1), xl, n);
    if (has_r) bs.add(st + nn + n * w + (n * w & 1) + n, xr, n);
    bulk_stage(bs, &bar, phase);
    for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) Ls[(idx / n) * ldl + idx % n] = st[idx];
    const double* Ws = st + nn;
    const double* xls = st + nn + n * w + (n * w & 1);
    const double* xrs = xls + n;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double t = 0.0;
      if (has_l)
        for (int c = 0; c < n; ++c) t += Ws[r * w + c] * xls[c];
      if (has_r)
        for (int c = 0; c < n; ++c) t += Ws[r * w + n + c] * xrs[c];
      v[r] = Ws[r * w + 2 * n] - t;
    }
  } else if (n > 64) {
    // The factor (row stride n + 2: 16-byte rows for the bulk copies; its
    // column reads below are at worst 4-way conflicted and every element is
    // read once) and the diagonal-block inverses come by bulk copies issued
    // up front, one memory latency overlapped with the v rows; v by one warp
    // per row with the lanes over the (coalesced) columns of W
    const int ldb = n + 2, nbk8 = (n + 7) / 8;
    double* Lsb = v + ((n + 16) & ~1);
    double* Lis = Lsb + (size_t)n * ldb;
    const double* Lig = L.Linv + (b * E + o) * nbk8 * 64;
    __shared__ __align__(8) uint64_t bbar;
    const bool tma = (n % 2) == 0;
    if (threadIdx.x == 0) mbar_init(&bbar, 1);
    __syncthreads();
    if (tma) {
      if (threadIdx.x < 32) {
        const int ln = threadIdx.x;
        fence_proxy_async();
        if (ln == 0) mbar_arrive_tx(&bbar, 8u * (uint32_t)(nn + nbk8 * 64));
        __syncwarp();
        for (int r = ln; r < n; r += 32) bulk_g2s(Lsb + (size_t)r * ldb, Lc + (size_t)r * n, 8u * n, &bbar);
        if (ln == 0) bulk_g2s(Lis, Lig, 8u * nbk8 * 64, &bbar);
      }
    } else {
      for (int idx = threadIdx.x; idx < nn; idx += blockDim.x) Lsb[(idx / n) * ldb + idx % n] = Lc[idx];
      for (int idx = threadIdx.x; idx < nbk8 * 64; idx += blockDim.x) Lis[idx] = Lig[idx];
    }
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // four rows of W per warp trip (independent loads, one latency for four rows)
    for (int r0 = threadIdx.x >> 5; r0 < n; r0 += 4 * nw) {
      double t[4] = {0.0, 0.0, 0.0, 0.0};
      for (int c = lane; c < n; c += 32) {
        const double xlc = has_l ? xl[c] : 0.0, xrc = has_r ? xr[c] : 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = r0 + e * nw;
          if (r < n) {
            if (has_l) t[e] += Wm[r * w + c] * xlc;
            if (has_r) t[e] += Wm[r * w + n + c] * xrc;
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = r0 + e * nw;
        const double ts = warp_sum(t[e]);
        if (lane == 0 && r < n) v[r] = Wm[r * w + 2 * n] - ts;
      }
    }
    if (tma) mbar_wait(&bbar, 0u);
  } else {
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double s = Wm[r * w + 2 * n];
      double t = 0.0;
      if (has_l)
        for (int c = 0; c < n; ++c) t += Wm[r * w + c] * xl[c];
      if (has_r)
        for (int c = 0; c < n; ++c) t += Wm[r * w + n + c] * xr[c];
      v[r] = s - t;
    }
  }
  __syncthreads();
  if (n <= 32) {
    // lane-per-row back substitution, x = L^{-T} v, one warp
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      double vi = lane < n ? v[lane] : 0.0;
      for (int r = n - 1; r >= 0; --r) {
        const double xr_ = __shfl_sync(0xffffffffu, vi / (lane == r ? Ls[r * ldl + r] : 1.0), r);
        if (lane == r) vi = xr_;
        if (lane < r) vi -= Ls[r * ldl + lane] * xr_;
      }
      if (lane < n) x[lane] = vi;
    }
    return;
  }
  if (n > 64) {
    // blocked x = L^{-T} v with the diagonal-block inverses of the split
    // elimination: per 8-row block, warp j reduces row k0 + j over the solved
    // rows, then x_k = Linv_k' r
    const int nbk = (n + 7) / 8, lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int ldb = n + 2;
    const double* Lsb = v + ((n + 16) & ~1);   // staged factor, stride n + 2
    const double* Li = Lsb + (size_t)n * ldb;   // staged diagonal-block inverses
    // right-looking: x_k = Linv_k' v_k by eight threads, then every unsolved
    // row j < k0 takes its rank-8 update v_j -= sum_i L[k0+i][j] x_{k0+i}
    // (thread per row, coalesced factor rows, no reductions) -- a quarter of
    // the left-looking step's latency (warp dot products over the solved rows)
    (void)lane;
    (void)wp;
    for (int kb = nbk - 1; kb >= 0; --kb) {
      const int k0 = kb * 8, rb = min(8, n - k0);
      if (threadIdx.x < 32) {
        double rr[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) rr[j] = j < rb ? v[k0 + j] : 0.0;
        __syncwarp();
        if (threadIdx.x < rb) {
          double xt = 0.0;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < rb) xt += Li[kb * 64 + j * 8 + threadIdx.x] * rr[j];
          v[k0 + threadIdx.x] = xt;
        }
      }
      __syncthreads();
      for (int j = threadIdx.x; j < k0; j += blockDim.x) {
        double t = v[j];
        for (int i = 0; i < rb; ++i) t -= Lsb[(k0 + i) * ldb + j] * v[k0 + i];
        v[j] = t;
      }
      __syncthreads();
    }
    for (int r = threadIdx.x; r < n; r += blockDim.x) x[r] = v[r];
    return;
  }
  const double* Lp = sm ? Ls : Lc;
  const int lp = sm ? ldl : n;
  for (int r = n - 1; r >= 0; --r) {
    if (threadIdx.x == 0) v[r] /= Lp[r * lp + r];
    __syncthreads();
    const double xr_ = v[r];
    for (int k = threadIdx.x; k < r; k += blockDim.x) v[k] -= Lp[r * lp + k] * xr_;
    __syncthreads();
  }
  for (int r = threadIdx.x; r < n; r += blockDim.x) x[r] = v[r];
}

// residual of the level-0 equations at the solved links (parallel.py:273-282):
// CTA i takes block row i, copies x_i out as link i and folds its maximum into
// link_residual[b] (zeroed by link_assemble0; the maximum of non-negative
// doubles = the maximum of their bit patterns, exact in any order)
__global__ void link_residual_part(plq_problem_t p, LinkLevel L, double* links, double* link_residual) {
  __shared__ double red[32];
  const int n = p.n, K = L.K;
  const int64_t nn = (int64_t)n * n;
  const int64_t b = blockIdx.x / K;
  const int i = blockIdx.x % K;
  const double* D = L.D + (b * K + i) * nn;
  const double* x = L.x + b * K * n;
  double worst = 0.0;
  if (n > 64) {
    // large blocks: the row products with lanes over the (coalesced) columns,
    // four rows per warp trip; the transposed term S_i' x_{i+1} thread per
    // column (coalesced across threads), staged in shared memory first
    __shared__ double tr[128];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool has_l = i >= 1, has_r = i + 1 < K;
    const double* Sl = has_l ? L.S + (b * (K - 1) + (i - 1)) * nn : nullptr;
    const double* Sr = has_r ? L.S + (b * (K - 1) + i) * nn : nullptr;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double t0 = 0.0, t1 = 0.0;
      if (has_r) {
        int c = 0;
        for (; c + 1 < n; c += 2) {
          t0 += Sr[c * n + r] * x[(i + 1) * n + c];
          t1 += Sr[(c + 1) * n + r] * x[(i + 1) * n + c + 1];
        }
        if (c < n) t0 += Sr[c * n + r] * x[(i + 1) * n + c];
      }
      tr[r] = t0 + t1;
    }
    __syncthreads();
    for (int r0 = wp; r0 < n; r0 += 4 * nw) {
      double t[4] = {0.0, 0.0, 0.0, 0.0};
      for (int c = lane; c < n; c += 32) {
        const double xi_ = x[i * n + c], xl_ = has_l ? x[(i - 1) * n + c] : 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = r0 + e * nw;
          if (r < n) {
            t[e] += D[r * n + c] * xi_;
            if (has_l) t[e] += Sl[r * n + c] * xl_;
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = r0 + e * nw;
        const double ts = warp_sum(t[e]);
        if (lane == 0 && r < n) worst = fmax(worst, fabs(ts + tr[r] - L.rhs[(b * K + i) * n + r]));
      }
    }
  } else {
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < n; ++c) s += D[r * n + c] * x[i * n + c];
    if (i >= 1) {
      const double* S = L.S + (b * (K - 1) + (i - 1)) * nn;
      for (int c = 0; c < n; ++c) s += S[r * n + c] * x[(i - 1) * n + c];
    }
    if (i + 1 < K) {
      const double* S = L.S + (b * (K - 1) + i) * nn;
      for (int c = 0; c < n; ++c) s += S[c * n + r] * x[(i + 1) * n + c];
    }
    worst = fmax(worst, fabs(s - L.rhs[(b * K + i) * n + r]));
  }
  }
  for (int r = threadIdx.x; r < n; r += blockDim.x) links[(b * K + i) * n + r] = x[i * n + r];
  worst = block_max(worst, red);
  if (threadIdx.x == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(link_residual + b), (unsigned long long)__double_as_longlong(worst));
}

int link_threads(int n) {
  if (n <= 16) return 32;
  if (n <= 32) return 128;
  return 256;
}

}  // namespace

size_t link_workspace_doubles(int64_t B, int J, int n) { return plan_link(B, J, n, nullptr).doubles; }

int launch_link_solve(const plq_problem_t& p, const double* vf0, double* links, double* link_residual,
                      int32_t* status, double* ws, cudaStream_t s, int* launches) {
  if (p.J < 2) return 0;
  LinkPlan P = plan_link(p.B, p.J, p.n, ws);
  const int threads = link_threads(p.n);
  const unsigned B = (unsigned)p.B;
  int nl = 0;
  // n <= 64: levels >= 1 assemble their own blocks inside the elimination (PLQ_LINK_FUSE=0: separate launches)
  const char* fe = getenv("PLQ_LINK_FUSE");
  const bool fuse = !(fe && fe[0] == '0') && p.n <= 64;
  const char* fs = getenv("PLQ_LINK_FSOLVE");   // 0: separate forward solve after the factorization (measurement)
  const int fsolve = !(fs && fs[0] == '0');
  link_assemble0<<<B * P.lv[0].K, p.n > 64 ? 1024 : threads, 0, s>>>(p, vf0, P.lv[0], link_residual);
  ++nl;
  for (size_t l = 0; l < P.lv.size(); ++l) {
    const int w = 2 * p.n + 1, ldw = ((w + 3) / 8) * 8 + 4;
    // the elimination is the level's critical path: 8 warps from n = 17 up
    const int ethreads = p.n <= 16 ? threads : 256;
    const bool esm = p.n <= 64, elsm = p.n <= 128;
    const int eldl = elsm ? p.n + 1 : p.n, eldw = esm ? ldw : w;
    const size_t tsm = sizeof(double) * (link_elim_blocked_off(p.n, esm, elsm, eldl, eldw, ethreads) +
                                         link_elim_blocked_doubles(p.n));
    if (p.n > 64) {
      const LinkLevel& Lv = P.lv[l];
      const int nbk = (p.n + 7) / 8, nt = (p.n + 63) / 64;
      const size_t fsm = sizeof(double) * (((size_t)p.n * link_ldl_big(p.n) + 1) / 2 * 2 + nbk * 64);
      const size_t rsm =
          sizeof(double) * ((size_t)p.n * link_ldl_big(p.n) + nbk * 64 + (size_t)p.n * LINK_SLAB_LD + 8 * 64);
      const size_t gsm = sizeof(double) * TileCfg<8>::DOUBLES;
      cudaFuncSetAttribute(link_factor_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
      cudaFuncSetAttribute(link_trsm_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
      if (gsm > 48 * 1024) cudaFuncSetAttribute(link_gram_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm);
      link_factor_big<<<B * Lv.E, 512, fsm, s>>>(p, Lv, status);
      link_trsm_big<<<B * Lv.E * link_slabs((int64_t)B * Lv.E), 256, rsm, s>>>(p, Lv, status);
      nl += 2;
      if (!Lv.top) {
        link_gram_big<<<B * Lv.E * (3 * nt * nt + 1), 256, gsm, s>>>(p, Lv, status);
        ++nl;
      }
    } else {
      const bool fl = l > 0 && fuse;
      const unsigned grid = B * (unsigned)(fl ? P.lv[l].K : P.lv[l].E);
      const bool deep = grid <= 148;   // one CTA per SM at most: no register cap
      auto kern = fl ? (deep ? link_eliminate<true, 1> : link_eliminate<true, 2>)
                     : (deep ? link_eliminate<false, 1> : link_eliminate<false, 2>);
      if (tsm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
      kern<<<grid, ethreads, tsm, s>>>(p, P.lv[l], fl ? P.lv[l - 1] : P.lv[l], status, fsolve);
      ++nl;
    }
    if (!P.lv[l].top && !fuse) {
      link_assemble_next<<<B * P.lv[l + 1].K, p.n > 64 ? 1024 : threads, 0, s>>>(p, P.lv[l], P.lv[l + 1]);
      ++nl;
    }
  }
  for (int l = (int)P.lv.size() - 1; l >= 0; --l) {
    const LinkLevel& C = P.lv[l + 1 < (int)P.lv.size() ? l + 1 : l];
    const size_t bsm = sizeof(double) * (p.n + 10 + (p.n <= 64 ? (size_t)p.n * (p.n + 1) + 4 + (size_t)p.n * p.n +
                                                              (size_t)p.n * (2 * p.n + 1) + 2 * p.n + 2
                                                          : (size_t)p.n * (p.n + 2) + (size_t)((p.n + 7) / 8) * 64 + 16));
    if (bsm > 48 * 1024) cudaFuncSetAttribute(link_backsub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    if (P.lv[l].top && p.n <= 64) continue;   // solved inside the top elimination
    link_backsub<<<B * P.lv[l].K, threads, bsm, s>>>(p, P.lv[l], C, l + 1 < (int)P.lv.size());
    ++nl;
  }
  link_residual_part<<<B * P.lv[0].K, threads, 0, s>>>(p, P.lv[0], links, link_residual);
  ++nl;
  if (launches) *launches += nl;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace plq
