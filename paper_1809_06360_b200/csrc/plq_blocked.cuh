// Blocked dense factorizations for a group of NWG warps (n, m >= 16):
// Cholesky, triangular solves and Householder QR in 8-wide blocks, so the
// sequential depth is m/8 block steps (two group barriers each) instead of m
// column steps, and the trailing work runs on the FP64 tensor pipe
// (DMMA.8x8x4, one 8 x 8 output tile per warp at a time).
//
// They replace the column-at-a-time cta_cholesky / cta_householder_qr /
// thread-per-column solves in the large-n sweeps and the link elimination
// (ncu source attribution on cfg4 put those at ~50 % of the sweep's stalls).
// The arithmetic is the same LAPACK-style algorithms (dpotrf, dtrsm, dgeqrf
// with dlarfg reflectors and the compact-WY dlarft/dlarfb update), blocked,
// so results agree with numpy/LAPACK to rounding.
//
// Conventions: row-major matrices with explicit leading dimensions, generic
// pointers (shared memory or global scratch).  `gt` is the thread index in
// the group, `sync()` the group barrier.  Every routine ends with a barrier.
// `wsc` is NWG * 64 doubles of per-warp scratch.
#pragma once

#include "plq_device.cuh"

namespace plq {

// ---------------------------------------------------------------------------
// Cholesky A = L L' (lower), block 8, right-looking.
//   * every thread that needs it factors the 8 x 8 diagonal block redundantly
//     in registers (ragged last block padded with the identity);
//   * threads t < below solve their panel row l = a L_kk^{-T}; threads
//     below <= t < below + 8 solve with unit rows, which yields the columns
//     of L_kk^{-1} (stored in Linv, block kb at Linv + 64 kb, row-major 8x8);
//   * the lower tiles of the trailing block get A -= l l' on DMMA.
// The strict upper triangle of A is left untouched; the DIAGONAL BLOCKS OF A
// ARE NOT OVERWRITTEN unless `Ld` (another nb * 64 doubles of staging) is
// given -- consumers use Linv for them.  Returns false (all threads) on a
// non-positive / NaN pivot (dpotrf failure).  `flag`: one int.
// With X (m x W, ldx) given, the forward solve X <- L^{-1} X is fused in:
// block row k of X is solved in step k's trailing phase, next to the Schur
// tiles (`wsc`: NWG * 64 doubles), which saves gtrsm8<0>'s m/8 barriers.
// Xsrc (optional, same stride) supplies the right-hand side instead of X's
// own contents, scaled by xscale: X <- L^{-1} (xscale * Xsrc) with no copy
// pass (block row k of Xsrc is read once, in step k).
// BATCH: the k-loops over already-solved rows of X load 8 k-steps of X before
// their DMMAs (X in L2 / DRAM scratch: a quarter of the latency exposures).
template <int NWG, bool BATCH = false, class Sync>
__device__ __forceinline__ bool gchol8(double* A, int m, int lda, double* Linv, int* flag, int gt, Sync sync,
                                       double* Ld = nullptr, double* X = nullptr, int W = 0, int ldx = 0,
                                       double* wsc = nullptr, const double* Xsrc = nullptr, double xscale = 1.0) {
  constexpr int NT = NWG * 32;
  const int lane = gt & 31, gw = gt >> 5, g = lane >> 2, q = lane & 3;
  for (int k0 = 0; k0 < m; k0 += 8) {
    const int rb = min(8, m - k0);
    const int below = m - k0 - rb;
    for (int t = gt; t < below + 8; t += NT) {
      double L[8][8], ri[8];
      bool ok = true;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int i = j; i < 8; ++i) {
          double v = (i < rb && j < rb) ? A[(k0 + i) * lda + k0 + j] : (i == j ? 1.0 : 0.0);
#pragma unroll
          for (int c = 0; c < j; ++c) v -= L[i][c] * L[j][c];
          if (i == j) {
            ok = ok && (v > 0.0);
            const double vv = v > 0.0 ? v : 1.0;
            const double rs = rsqrt(vv);
            L[j][j] = vv * rs;
            ri[j] = rs;
          } else {
            L[i][j] = v * ri[j];
          }
        }
      }
      // row vector a: a panel row of A, or the unit row e_u (-> column u of L^{-1})
      const bool panel = t < below;
      const int u = t - below;
      double a[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        a[c] = panel ? (c < rb ? A[(k0 + rb + t) * lda + k0 + c] : 0.0) : (c == u ? 1.0 : 0.0);
      // solve L x = a' (forward substitution)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double v = a[j];
#pragma unroll
        for (int c = 0; c < j; ++c) v -= L[j][c] * a[c];
        a[j] = v * ri[j];
      }
      if (panel) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < rb) A[(k0 + rb + t) * lda + k0 + c] = a[c];
      } else {
        double* Li = Linv + (k0 >> 3) * 64;
#pragma unroll
        for (int i = 0; i < 8; ++i) Li[i * 8 + u] = a[i];
        if (Ld != nullptr && u == 0) {
          double* Lk = Ld + (k0 >> 3) * 64;
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) Lk[i * 8 + j] = (j <= i) ? L[i][j] : 0.0;
        }
      }
      if (t == 0) *flag = ok ? 0 : 1;
    }
    sync();
    if (*flag) {
      sync();
      return false;
    }
    // trailing update of the lower tiles: A[i][j] -= sum_c l_ic l_jc, and
    // (fused solve) block row k of X
    const int r0 = k0 + rb;
    const int tt = (below + 7) >> 3;
    const int nschur = tt * (tt + 1) / 2, nrhs = X != nullptr ? (W + 7) >> 3 : 0;
    for (int t = gw; t < nschur + nrhs; t += NWG) {
      if (t < nschur) continue;
      // X_k = Linv_kk (X_k - sum_{c < k0} L[k][c] X_c)
      double* ws = wsc + gw * 64;
      const double* D = Linv + (k0 >> 3) * 64;
      const int j0 = (t - nschur) * 8;
      double c0 = 0.0, c1 = 0.0;
      if constexpr (BATCH) {
        for (int kk0 = 0; kk0 < k0; kk0 += 32) {
          double bvs[8];
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int k = kk0 + 4 * ks + q;
            bvs[ks] = (k < k0 && j0 + g < W) ? X[k * ldx + j0 + g] : 0.0;
          }
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int k = kk0 + 4 * ks + q;
            dmma884(c0, c1, (k < k0 && g < rb) ? A[(k0 + g) * lda + k] : 0.0, bvs[ks]);
          }
        }
      } else {
#pragma unroll 4
        for (int kk = 0; kk < k0; kk += 4) {
          const int k = kk + q;
          const double av = (g < rb) ? A[(k0 + g) * lda + k] : 0.0;
          const double bv = (j0 + g < W) ? X[k * ldx + j0 + g] : 0.0;
          dmma884(c0, c1, av, bv);
        }
      }
      const int j = j0 + 2 * q;
      const double* Xs = Xsrc != nullptr ? Xsrc : X;
      ws[g * 8 + 2 * q] = (g < rb && j < W) ? xscale * Xs[(k0 + g) * ldx + j] - c0 : 0.0;
      ws[g * 8 + 2 * q + 1] = (g < rb && j + 1 < W) ? xscale * Xs[(k0 + g) * ldx + j + 1] - c1 : 0.0;
      __syncwarp();
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const int k = kk + q;
        dmma884(d0, d1, D[g * 8 + k], ws[k * 8 + g]);
      }
      if (g < rb) {
        if (j < W) X[(k0 + g) * ldx + j] = d0;
        if (j + 1 < W) X[(k0 + g) * ldx + j + 1] = d1;
      }
      __syncwarp();
    }
    for (int tile = gw; tile < nschur; tile += NWG) {
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
      const int tj = tile - ti * (ti + 1) / 2;
      const int i = r0 + ti * 8 + g, jb = r0 + tj * 8;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const int k = kk + q;
        const double av = (i < m && k < rb) ? A[i * lda + k0 + k] : 0.0;
        const double bv = (jb + g < m && k < rb) ? A[(jb + g) * lda + k0 + k] : 0.0;
        dmma884(c0, c1, av, bv);
      }
      const int j0 = jb + 2 * q;
      if (i < m) {
        if (j0 < m && (ti != tj || j0 <= i)) A[i * lda + j0] -= c0;
        if (j0 + 1 < m && (ti != tj || j0 + 1 <= i)) A[i * lda + j0 + 1] -= c1;
      }
    }
    sync();
  }
  if (Ld != nullptr) {
    // diagonal blocks (lower, with the diagonal) into A
    constexpr int NT = NWG * 32;
    for (int e = gt; e < ((m + 7) >> 3) * 64; e += NT) {
      const int kb = e >> 6, i = (e >> 3) & 7, j = e & 7, r = kb * 8 + i, c = kb * 8 + j;
      if (j <= i && r < m) A[r * lda + c] = Ld[e];
    }
    sync();
  }
  return true;
}

// Inverses of the 8 x 8 diagonal blocks of an upper-triangular R (m x m,
// diagonal taken from rdiag): block kb at Rinv + 64 kb (row-major, upper).
// Thread (kb, u) back-substitutes the unit column e_u.
template <int NWG, class Sync>
__device__ __forceinline__ void gtri_inv_upper8(const double* R, int m, int ldr, const double* rdiag, double* Rinv,
                                                int gt, Sync sync) {
  constexpr int NT = NWG * 32;
  const int nb = (m + 7) >> 3;
  for (int t = gt; t < nb * 8; t += NT) {
    const int kb = t >> 3, u = t & 7, k0 = kb * 8, rb = min(8, m - k0);
    double x[8];
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      double v = (i == u) ? 1.0 : 0.0;
#pragma unroll
      for (int c = i + 1; c < 8; ++c)
        if (c < rb && i < rb) v -= R[(k0 + i) * ldr + k0 + c] * x[c];
      x[i] = (i < rb) ? v / rdiag[k0 + i] : v;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) Rinv[kb * 64 + i * 8 + u] = x[i];
  }
  sync();
}

// Blocked triangular solve on an m x W block X (ldx), in place, by 8-row
// block steps; in each step warp-owned 8 x 8 column tiles compute
//   R = X_k - sum_{c in done} T(k, c) X_c     (DMMA over the finished rows)
//   X_k = D_k R                                (DMMA with the block inverse)
// MODE 0: L x = b (L lower, forward; T(k,c) = L[k][c], D = Linv)
// MODE 1: L' x = b (backward; T(k,c) = L[c][k], D = Linv')
// MODE 2: R x = b (R upper, backward; T(k,c) = R[k][c], D = Rinv)
template <int MODE, int NWG, bool BATCH = false, class Sync>
__device__ __forceinline__ void gtrsm8(const double* T, int m, int ldt, const double* Dinv, double* X, int W, int ldx,
                                       double* wsc, int gt, Sync sync) {
  const int lane = gt & 31, gw = gt >> 5, g = lane >> 2, q = lane & 3;
  const int nb = (m + 7) >> 3, tn = (W + 7) >> 3;
  double* ws = wsc + gw * 64;
  for (int step = 0; step < nb; ++step) {
    const int kb = (MODE == 0) ? step : nb - 1 - step;
    const int k0 = kb * 8, rb = min(8, m - k0);
    const double* D = Dinv + kb * 64;
    // finished rows: [0, k0) forward, [k0 + rb, m) backward
    const int c_lo = (MODE == 0) ? 0 : k0 + rb, c_hi = (MODE == 0) ? k0 : m;
    for (int tj = gw; tj < tn; tj += NWG) {
      const int j0 = tj * 8;
      double c0 = 0.0, c1 = 0.0;
      if constexpr (BATCH) {
        for (int kk0 = c_lo; kk0 < c_hi; kk0 += 32) {
          double bvs[8];
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int k = kk0 + 4 * ks + q;
            bvs[ks] = (k < c_hi && j0 + g < W) ? X[k * ldx + j0 + g] : 0.0;
          }
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int k = kk0 + 4 * ks + q;
            const int i = k0 + g;
            double av = 0.0;
            if (k < c_hi && g < rb) av = (MODE == 1) ? T[k * ldt + i] : T[i * ldt + k];
            dmma884(c0, c1, av, bvs[ks]);
          }
        }
      } else {
#pragma unroll 4
        for (int kk = c_lo; kk < c_hi; kk += 4) {
          const int k = kk + q;
          const bool kv = k < c_hi;
          const int i = k0 + g;
          double av = 0.0;
          if (kv && g < rb) av = (MODE == 1) ? T[k * ldt + i] : T[i * ldt + k];
          const double bv = (kv && j0 + g < W) ? X[k * ldx + j0 + g] : 0.0;
          dmma884(c0, c1, av, bv);
        }
      }
      // R tile (rows g < rb of block k, columns j0 + 2q + e) -> warp scratch
      const int j = j0 + 2 * q;
      ws[g * 8 + 2 * q] = (g < rb && j < W) ? X[(k0 + g) * ldx + j] - c0 : 0.0;
      ws[g * 8 + 2 * q + 1] = (g < rb && j + 1 < W) ? X[(k0 + g) * ldx + j + 1] - c1 : 0.0;
      __syncwarp();
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const int k = kk + q;
        const double av = (MODE == 1) ? D[k * 8 + g] : D[g * 8 + k];
        dmma884(d0, d1, av, ws[k * 8 + g]);
      }
      if (g < rb) {
        if (j < W) X[(k0 + g) * ldx + j] = d0;
        if (j + 1 < W) X[(k0 + g) * ldx + j + 1] = d1;
      }
      __syncwarp();
    }
    sync();
  }
}

// Householder QR of the r x M panel A (lda), Q' applied to the r x W block X
// (ldx), in 8-column panels: warp 0 factors the panel (dlarfg reflectors,
// LAPACK convention R_jj = beta, v_j = 1), forms T (dlarft, forward
// columnwise, Q_p = I - V T V') and VT = V T'; then every warp applies
// Q_p' = I - V T' V' to its 8-column tiles of [A(:, p0+8:M) | X] as
// Y = V' C (DMMA, K = r - p0) and C -= VT Y (DMMA, K = 8).
// On exit A holds R (upper) and V (strictly lower), rdiag = diag(R).
// Scratch: Tm 64 doubles, VT r * 8 doubles, wsc NWG * 64.
// RS > 0: warp 0 holds the panel in registers (row li = lane + 32 s, s < RS;
// needs r <= 32 RS) and batches the independent warp reductions of each
// column step; RS = 0: the panel stays in memory (any r, fewer registers).
template <int N8>
__device__ __forceinline__ void warp_sum_batch(double (&v)[N8]) {
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int k = 0; k < N8; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}

// TS != nullptr keeps T (8 x 8) in shared memory instead of registers (for
// register-capped 16-warp CTAs).
// VS != nullptr: the reflectors V (rows x 8, explicit unit diagonal / zeros)
// are also stored there, so the trailing update reads them from shared memory.
template <int RS>
__device__ __forceinline__ void qr_panel_regs(double* A, int lda, int p0, int pb, int rows, double* rdiag,
                                              double* VT, int lane, double* TS = nullptr, double* VS = nullptr) {
  double a[RS][8];
#pragma unroll
  for (int s = 0; s < RS; ++s)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int li = lane + 32 * s;
      a[s][c] = (li < rows && c < pb) ? A[(p0 + li) * lda + p0 + c] : 0.0;
    }
  double tau[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    tau[j] = 0.0;
    if (j < pb) {
      double part = 0.0;
#pragma unroll
      for (int s = 0; s < RS; ++s) part += (lane + 32 * s > j) ? a[s][j] * a[s][j] : 0.0;
      const double sig = warp_sum(part);
      const double alpha = __shfl_sync(0xffffffffu, a[0][j], j);
      double t = 0.0, beta = alpha, scale = 0.0;
      if (sig > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sig), alpha);
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      tau[j] = t;
      double v[RS];
#pragma unroll
      for (int s = 0; s < RS; ++s) {
        const int li = lane + 32 * s;
        v[s] = (li == j) ? 1.0 : (li > j ? a[s][j] * scale : 0.0);
      }
      // H_j applied to the columns k > j: a_k -= t v (v' a_k), all sums at once
      double pk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        pk[k] = 0.0;
        if (k > j) {
#pragma unroll
          for (int s = 0; s < RS; ++s) pk[k] += v[s] * a[s][k];
        }
      }
      warp_sum_batch(pk);
#pragma unroll
      for (int k = j + 1; k < 8; ++k)
#pragma unroll
        for (int s = 0; s < RS; ++s) a[s][k] -= t * pk[k] * v[s];
#pragma unroll
      for (int s = 0; s < RS; ++s) {
        const int li = lane + 32 * s;
        if (li > j) a[s][j] = v[s];
        if (li == j) a[s][j] = beta;
      }
      if (lane == 0) rdiag[p0 + j] = beta;
    }
  }
  // T (upper): T_jj = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] (V' v_j)[0:j]
  double Tr[8][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      w[i] = 0.0;
      if (i < j) {
#pragma unroll
        for (int s = 0; s < RS; ++s) {
          const int li = lane + 32 * s;
          const double vi = (li == i) ? 1.0 : (li > i ? a[s][i] : 0.0);
          const double vj = (li == j) ? 1.0 : (li > j ? a[s][j] : 0.0);
          w[i] += vi * vj;
        }
      }
    }
    warp_sum_batch(w);
    if (TS != nullptr) {
      double col[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double sacc = 0.0;
        if (i < j) {
#pragma unroll
          for (int k = i; k < j; ++k) sacc += TS[i * 8 + k] * w[k];
        }
        col[i] = (i < j) ? -tau[j] * sacc : (i == j ? tau[j] : 0.0);
      }
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) TS[i * 8 + j] = col[i];
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) Tr[i][j] = 0.0;
      Tr[j][j] = tau[j];
#pragma unroll
      for (int i = 0; i < j; ++i) {
        double sacc = 0.0;
#pragma unroll
        for (int k = i; k < j; ++k) sacc += Tr[i][k] * w[k];
        Tr[i][j] = -tau[j] * sacc;
      }
    }
  }
#pragma unroll
  for (int s = 0; s < RS; ++s) {
    const int li = lane + 32 * s;
    if (li < rows) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < pb) A[(p0 + li) * lda + p0 + c] = a[s][c];
      double v[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) v[l] = (l >= pb || li < l) ? 0.0 : (li == l ? 1.0 : a[s][l]);
      if (VS != nullptr) {
#pragma unroll
        for (int l = 0; l < 8; ++l) VS[li * 8 + l] = v[l];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double sacc = 0.0;
#pragma unroll
        for (int l = c; l < 8; ++l) sacc += v[l] * (TS != nullptr ? TS[c * 8 + l] : Tr[c][l]);
        VT[li * 8 + c] = sacc;
      }
    }
  }
}

template <int NWG, class Sync, int RS = 0>
__device__ __forceinline__ void gqr8(double* A, int r, int M, int lda, double* X, int W, int ldx, double* rdiag,
                                     double* VT, double* wsc, int gt, Sync sync, double* TS = nullptr,
                                     double* VS = nullptr) {
  const int lane = gt & 31, gw = gt >> 5, g = lane >> 2, q = lane & 3;
  double* ws = wsc + gw * 64;
  for (int p0 = 0; p0 < M; p0 += 8) {
    const int pb = min(8, M - p0);
    const int rows = r - p0;   // panel rows p0 .. r-1 (local index li)
    if constexpr (RS > 0) {
      if (gw == 0) qr_panel_regs<RS>(A, lda, p0, pb, rows, rdiag, VT, lane, TS, VS);
    } else if (gw == 0) {
      double tau[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        tau[j] = 0.0;
        if (j < pb) {
          double part = 0.0;
          for (int li = j + 1 + lane; li < rows; li += 32) {
            const double v = A[(p0 + li) * lda + p0 + j];
            part += v * v;
          }
          const double sig = warp_sum(part);
          const double alpha = A[(p0 + j) * lda + p0 + j];
          double t = 0.0, beta = alpha, scale = 0.0;
          if (sig > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + sig), alpha);
            t = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
          }
          tau[j] = t;
          for (int li = j + 1 + lane; li < rows; li += 32) A[(p0 + li) * lda + p0 + j] *= scale;
          __syncwarp();
          // apply H_j to the panel's remaining columns k > j: a_k -= t v (v' a_k)
#pragma unroll
          for (int k = j + 1; k < 8; ++k) {
            if (k < pb) {
              double s = 0.0;
              for (int li = j + 1 + lane; li < rows; li += 32)
                s += A[(p0 + li) * lda + p0 + j] * A[(p0 + li) * lda + p0 + k];
              s = warp_sum(s) + A[(p0 + j) * lda + p0 + k];
              s *= t;
              __syncwarp();
              for (int li = j + 1 + lane; li < rows; li += 32)
                A[(p0 + li) * lda + p0 + k] -= s * A[(p0 + li) * lda + p0 + j];
              if (lane == 0) A[(p0 + j) * lda + p0 + k] -= s;
              __syncwarp();
            }
          }
          if (lane == 0) {
            A[(p0 + j) * lda + p0 + j] = beta;
            rdiag[p0 + j] = beta;
          }
          __syncwarp();
        }
      }
      // T (upper, pb x pb): T_jj = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] (V' v_j)[0:j]
      double Tr[8][8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = 0.0;
#pragma unroll
        for (int i = 0; i < j; ++i) {
          if (j >= pb) break;
          // (V' v_j)_i = sum_l v_i(l) v_j(l), v_i(l) = 0 for l < i, 1 at l = i
          double s = 0.0;
          for (int li = j + lane; li < rows; li += 32) {
            const double vj = (li == j) ? 1.0 : A[(p0 + li) * lda + p0 + j];
            s += A[(p0 + li) * lda + p0 + i] * vj;   // li >= j > i: v_i(li) is stored
          }
          w[i] = warp_sum(s);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) Tr[i][j] = 0.0;
        Tr[j][j] = tau[j];
#pragma unroll
        for (int i = 0; i < j; ++i) {
          double s = 0.0;
#pragma unroll
          for (int k = i; k < j; ++k) s += Tr[i][k] * w[k];
          Tr[i][j] = -tau[j] * s;
        }
      }
      // VT = V T' (rows li, 8 columns): (V T')_{li, c} = sum_{l >= c} v_l(li) T[c][l]
      for (int li = lane; li < rows; li += 32) {
        double v[8];
#pragma unroll
        for (int l = 0; l < 8; ++l)
          v[l] = (l >= pb || li < l) ? 0.0 : (li == l ? 1.0 : A[(p0 + li) * lda + p0 + l]);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double s = 0.0;
#pragma unroll
          for (int l = c; l < 8; ++l) s += v[l] * Tr[c][l];
          VT[li * 8 + c] = s;
        }
      }
    }
    sync();
    // trailing update of C = [A(:, p0+pb : M) | X], rows p0 .. r-1
    const int na = (M - p0 - pb + 7) >> 3, nx = (W + 7) >> 3;
    for (int t = gw; t < na + nx; t += NWG) {
      double* C;
      int ldc, ncol;
      if (t < na) {
        C = A + p0 * lda + p0 + pb + t * 8;
        ldc = lda;
        ncol = min(8, M - p0 - pb - t * 8);
      } else {
        C = X + p0 * ldx + (t - na) * 8;
        ldc = ldx;
        ncol = min(8, W - (t - na) * 8);
      }
      // Y = V' C (8 x 8, K = rows): V'(i, l) = v_i(l)
      double y0 = 0.0, y1 = 0.0;
      if constexpr (RS > 0 && RS <= 2) {
        // rows <= 64: every C load of the tile issued up front (C may live in
        // L2 scratch: one latency exposure instead of one per 4 k-steps)
        constexpr int KS = 8 * RS;
        double avs[KS], bvs[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int l = 4 * ks + q;
          avs[ks] = (l < rows && g < pb) ? ((l == g) ? 1.0 : (l > g ? A[(p0 + l) * lda + p0 + g] : 0.0)) : 0.0;
          bvs[ks] = (l < rows && g < ncol) ? C[l * ldc + g] : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) dmma884(y0, y1, avs[ks], bvs[ks]);
      } else if (VS != nullptr) {
        // any row count: C (L2 / DRAM scratch) loaded 8 k-steps at a time
        // before their DMMAs -- a quarter of the latency exposures of a
        // load-per-step loop; the reflectors come from shared memory
        for (int kk0 = 0; kk0 < rows; kk0 += 32) {
          double bvs[8];
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int l = kk0 + 4 * ks + q;
            bvs[ks] = (l < rows && g < ncol) ? C[l * ldc + g] : 0.0;
          }
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int l = kk0 + 4 * ks + q;
            dmma884(y0, y1, l < rows ? VS[l * 8 + g] : 0.0, bvs[ks]);
          }
        }
      } else {
#pragma unroll 4
        for (int kk = 0; kk < rows; kk += 4) {
          const int l = kk + q;
          double av = 0.0;
          if (l < rows && g < pb) av = (l == g) ? 1.0 : (l > g ? A[(p0 + l) * lda + p0 + g] : 0.0);
          const double bv = (l < rows && g < ncol) ? C[l * ldc + g] : 0.0;
          dmma884(y0, y1, av, bv);
        }
      }
      ws[g * 8 + 2 * q] = y0;
      ws[g * 8 + 2 * q + 1] = y1;
      __syncwarp();
      // C -= VT Y, 8-row bands
      if constexpr (RS > 0 && RS <= 2) {
        constexpr int NB = 4 * RS;   // 8-row bands of <= 32 RS rows
        const int j = 2 * q;
        double cur[NB][2];
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) {   // loads first (L2 latency once)
          const int i = bb * 8 + g;
          cur[bb][0] = (i < rows && j < ncol) ? C[i * ldc + j] : 0.0;
          cur[bb][1] = (i < rows && j + 1 < ncol) ? C[i * ldc + j + 1] : 0.0;
        }
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int kk = 0; kk < 8; kk += 4) {
            const int k = kk + q;
            const double av = (bb * 8 + g < rows) ? VT[(bb * 8 + g) * 8 + k] : 0.0;
            dmma884(c0, c1, av, ws[k * 8 + g]);
          }
          const int i = bb * 8 + g;
          if (i < rows) {
            if (j < ncol) C[i * ldc + j] = cur[bb][0] - c0;
            if (j + 1 < ncol) C[i * ldc + j + 1] = cur[bb][1] - c1;
          }
        }
      } else if (VS != nullptr) {
        const int j = 2 * q;
        for (int b00 = 0; b00 < rows; b00 += 32) {   // four 8-row bands: loads first
          double cur[4][2];
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const int i = b00 + bb * 8 + g;
            cur[bb][0] = (i < rows && j < ncol) ? C[i * ldc + j] : 0.0;
            cur[bb][1] = (i < rows && j + 1 < ncol) ? C[i * ldc + j + 1] : 0.0;
          }
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const int i = b00 + bb * 8 + g;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; kk += 4) {
              const int k = kk + q;
              dmma884(c0, c1, i < rows ? VT[i * 8 + k] : 0.0, ws[k * 8 + g]);
            }
            if (i < rows) {
              if (j < ncol) C[i * ldc + j] = cur[bb][0] - c0;
              if (j + 1 < ncol) C[i * ldc + j + 1] = cur[bb][1] - c1;
            }
          }
        }
      } else {
#pragma unroll 2
        for (int b0 = 0; b0 < rows; b0 += 8) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int kk = 0; kk < 8; kk += 4) {
            const int k = kk + q;
            const double av = (b0 + g < rows) ? VT[(b0 + g) * 8 + k] : 0.0;
            dmma884(c0, c1, av, ws[k * 8 + g]);
          }
          const int i = b0 + g, j = 2 * q;
          if (i < rows) {
            if (j < ncol) C[i * ldc + j] -= c0;
            if (j + 1 < ncol) C[i * ldc + j + 1] -= c1;
          }
        }
      }
      __syncwarp();
    }
    sync();
  }
}

}  // namespace plq
