// K1: per-segment backward sweeps of the horizon-partitioned Riccati solve.
//
// One CTA owns one segment of one problem and walks its stages backwards.
//   * endpoint segments (j < J-1): endpoint-explicit sweep with zero terminal
//     cost and terminal rows Hx=I, Hz=-I -- endpoint.backward_pass
//     (/root/reference/pkg/src/parlqr/endpoint.py:168-301) as called by
//     parallel._solve_segment_task (parallel.py:228-240);
//   * the last segment: plain Riccati sweep from the terminal cost --
//     serial.backward_pass (serial.py:37-79).
//
// Per stage, with F = [Fx | Fu | f1]:
//   GEMM1  [VF; Z] = [Vxx; Vzx] F            (+ vx1 / vz1 in the last column)
//   GEMM2  [Mxx mx1; Mux Muu mu1] = [Fx Fu]' VF + Q-blocks
//   gains  G = [Kx | Kz | k1]:  r = 0: G = -Muu^{-1} [Mux | Mzu' | mu1]
//          tail (r >= m): Householder QR of Nu = Hx Fu replaces the SVD of
//          endpoint.py:226 -- G = -R^{-1} Q1' [Nx Nz n1], rows <- Q2'[Nx Nz n1]
//          (pinv, projector and compressed rows are invariant to the row
//          basis); 0 < r < m: mixed range/null branch.
//   value  Y = P + Muu G;  [Vxx Vzx' vx1; Vzx Vzz vz1] = M + P'G + G'Y
//          which is term-for-term endpoint.py:285-294.
#pragma once
#include "plq_blocked.cuh"
#include "plq_device.cuh"
#include "plq_gemm.cuh"
#include "plq_internal.h"
#include "plq_rank.cuh"
#include "plq_tma.cuh"

#include <algorithm>

namespace plq {

namespace {

// Optional per-phase cycle accounting of the generic sweep (measurement build
// -DPLQ_PHASE_PROFILE only): thread 0 of every CTA adds clock64() deltas per
// stage phase into g_gen_phase[blockIdx.x][phase].
#ifdef PLQ_PHASE_PROFILE
__device__ unsigned long long g_gen_phase[1024][16];
#define PLQ_GPH(k)                                                                              \
  do {                                                                                          \
    if (threadIdx.x == 0) {                                                                     \
      const long long t_ = clock64();                                                           \
      atomicAdd(&g_gen_phase[blockIdx.x & 1023][k], (unsigned long long)(t_ - t_last));         \
      t_last = t_;                                                                              \
    }                                                                                           \
  } while (0)
#else
#define PLQ_GPH(k) \
  do {             \
  } while (0)
#endif

struct Bufs {
  double *V, *IN, *PGY, *MUU, *MISC, *VF, *Z, *MX, *H, *WIDE;
  double* tiles;   // tiled-GEMM staging (large mode) or nullptr
};

// large GEMMs go through the tiled DMMA kernel when the operands live in
// global scratch (large mode), small ones through the direct-fragment GEMM
template <bool TA, int NT, class Epi>
__device__ __forceinline__ void gemm_x(int M, int N, int K, const double* A, int lda, const double* B, int ldb,
                                       double* tiles, Epi epi) {
  if constexpr (NT >= 256) {
    if (tiles != nullptr && (long long)M * N * K >= 16384) {
      cta_gemm_tiled<TA, NT / 32, Epi, false, NoPre, sweep_tile_stages(NT)>(M, N, K, A, lda, B, ldb, tiles, epi);
      return;
    }
  }
  cta_gemm<TA, false, 1, 1>(M, N, K, A, lda, B, ldb, epi);
}

// gemm_x with an addend pre(i, j) loaded before the k-loop (epi gets pre + acc)
template <bool TA, int NT, class Pre, class Epi>
__device__ __forceinline__ void gemm_x_pre(int M, int N, int K, const double* A, int lda, const double* B, int ldb,
                                           double* tiles, Pre pre, Epi epi) {
  if constexpr (NT >= 256) {
    if (tiles != nullptr && (long long)M * N * K >= 16384) {
      cta_gemm_tiled<TA, NT / 32, Epi, true, Pre, sweep_tile_stages(NT)>(M, N, K, A, lda, B, ldb, tiles, epi, pre);
      return;
    }
  }
  cta_gemm<TA, false, 1, 1>(M, N, K, A, lda, B, ldb, [&](int i, int j, double acc) { epi(i, j, pre(i, j) + acc); });
}

// Symmetric result C = pre + op(A) B (Mxx = Qxx + Fx' VFx, Vxx += P'G): in
// large mode only the tiles on / below the diagonal are computed and the
// epilogue mirrors (i, j <= i) into (j, i), so C is exactly symmetric and no
// symmetrization pass is needed (what the n = 64 kernel does); returns false
// when the shape takes the direct path (caller symmetrizes as before).
template <bool TA, int NT, class Pre, class Epi>
__device__ __forceinline__ bool gemm_x_pre_sym(int N, int K, const double* A, int lda, const double* B, int ldb,
                                               double* tiles, Pre pre, Epi epi) {
  if constexpr (NT >= 256) {
    if (tiles != nullptr && (long long)N * N * K >= 16384) {
      cta_gemm_tiled<TA, NT / 32, Epi, true, Pre, sweep_tile_stages(NT), true>(N, N, K, A, lda, B, ldb, tiles, epi, pre);
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ void cho_solve_x(const double* L, int m, int ldl, double* X, int W, int ldx) {
  if (m >= 16)
    cta_cho_solve_blocked(L, m, ldl, X, W, ldx);
  else
    cta_cho_solve(L, m, ldl, X, W, ldx);
}

__device__ int wide_branch(const plq_problem_t& p, int n, int m, int r, int W, int ldw, int Fw, double* VF,
                            double* H, double* P, double* G, double* Muu, double* WIDE, double* tau, double* rdiag,
                            double* red, int* iflag, double thr_scale, int* status_out, int stage) {
  // Mixed branch 0 < p = r < m (endpoint.py:234-250): Nu (r x m) has full
  // row rank.  QR of Nu' = Q [R; 0]; pinv(Nu) = Q1 R^{-T}; null basis Q2.
  const int tid = threadIdx.x, nt = blockDim.x;
  double* X = WIDE;              // m x r   (Nu')
  double* Qm = X + m * r;        // m x m   (Q' Muu Q)
  double* BASE = Qm + m * m;     // m x ldw
  double* C = BASE + m * ldw;    // m x ldw
  for (int idx = tid; idx < m * r; idx += nt) {
    const int c = idx / r, i = idx % r;
    X[c * r + i] = VF[i * Fw + n + c];
  }
  __syncthreads();
  cta_householder_qr(X, m, r, r, nullptr, 0, 1, tau, rdiag, red);
  // rank certificates (plq_rank.cuh): ||Rw||_F <= thr -> p = 0 for sure;
  // 1 / ||Rw^{-1}||_F > thr -> p = r for sure; otherwise the SVD decides
  double rmax = 0.0, pf = 0.0, pi = 0.0;
  for (int i = 0; i < r; ++i) rmax = fmax(rmax, fabs(rdiag[i]));
  for (int idx = tid; idx < r * r; idx += nt) {
    const int i = idx / r, c = idx % r;
    if (c > i) pf += X[i * r + c] * X[i * r + c];
    if (c == i) pf += rdiag[i] * rdiag[i];
  }
  for (int c = tid; c < r; c += nt) {   // column c of Rw^{-1} into BASE (free here)
    for (int i = c; i >= 0; --i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int k = i + 1; k <= c; ++k) v -= X[i * r + k] * BASE[k * ldw + c];
      v /= rdiag[i];
      BASE[i * ldw + c] = v;
      pi += v * v;
    }
  }
  const double rf2 = block_sum(pf, red);
  const double ri2 = block_sum(pi, red);
  const double thr = p.rank_tol * fmax(thr_scale, rmax);
  if (sqrt(rf2) <= thr) return 1;                 // p = 0: Cholesky gains, all rows stay
  if (!(ri2 * thr * thr < 1.0)) return 2;         // undecided: rank-revealing path
  // y = R^{-T} stack (forward substitution), BASE = Q [y; 0]
  for (int c = tid; c < W; c += nt) {
    for (int i = 0; i < r; ++i) {
      double s = H[i * ldw + c];
      for (int k = 0; k < i; ++k) s -= X[k * r + i] * BASE[k * ldw + c];
      BASE[i * ldw + c] = s / rdiag[i];
    }
    for (int i = r; i < m; ++i) BASE[i * ldw + c] = 0.0;
  }
  __syncthreads();
  cta_apply_q(X, m, r, r, tau, BASE, W, ldw, true);
  // C = P - Muu BASE
  cta_gemm<false, false, 1, 1>(m, W, m, Muu, m, BASE, ldw,
                               [&](int i, int j, double acc) { C[i * ldw + j] = P[i * ldw + j] - acc; });
  // Qm = Muu, then Q' Muu, transpose, Q' (Muu Q) -> Q' Muu Q
  for (int idx = tid; idx < m * m; idx += nt) Qm[idx] = Muu[idx];
  __syncthreads();
  cta_apply_q(X, m, r, r, tau, Qm, m, m, false);
  for (int idx = tid; idx < m * m; idx += nt) {
    const int i = idx / m, j = idx % m;
    if (i < j) {
      const double a = Qm[i * m + j];
      Qm[i * m + j] = Qm[j * m + i];
      Qm[j * m + i] = a;
    }
  }
  __syncthreads();
  cta_apply_q(X, m, r, r, tau, Qm, m, m, false);
  cta_apply_q(X, m, r, r, tau, C, W, ldw, false);   // C <- Q' C
  // chol of W = Q2' Muu Q2 (the (m-r) x (m-r) trailing block)
  const int q = m - r;
  double* Wn = Qm + r * m + r;
  if (tid == 0) *iflag = 0;
  __syncthreads();
  if (!cta_cholesky(Wn, q, m, iflag)) {
    if (tid == 0) *status_out = 1 + stage;
    __syncthreads();
    return -1;
  }
  cta_cho_solve(Wn, q, m, C + r * ldw, W, ldw);
  for (int idx = tid; idx < r * W; idx += nt) C[(idx / W) * ldw + idx % W] = 0.0;
  __syncthreads();
  cta_apply_q(X, m, r, r, tau, C, W, ldw, true);   // Q [0; x]
  for (int idx = tid; idx < m * W; idx += nt) {
    const int i = idx / W, j = idx % W;
    G[i * ldw + j] = -(BASE[i * ldw + j] + C[i * ldw + j]);
  }
  __syncthreads();
  return 0;
}

template <int NT, bool REPAIR>
__device__ void sweep_segment(const SweepArgs& a, const Bufs& bf, int64_t b, int j) {
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, J = p.J, T = p.T;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lo = p.split_times[j], hi = p.split_times[j + 1], L = hi - lo;
  const bool serial = (j == J - 1 && !a.endpoint_terminal) || a.smooth_vf0;
  const int nz = serial ? 0 : n;
  const int cc = n + nz;            // constant column of G
  const int W = cc + 1;             // logical width of P/G/Y
  // storage strides of P/G/Y/H and of F/VF/Z (logical width n+m+1): even in
  // large mode, so the tiled GEMM streams its operands with 16-byte copies
  const int ldw = a.lay.large ? 2 * n + 2 : 2 * n + 1;
  const int Fw = a.lay.large ? ((n + m + 2) & ~1) : n + m + 1;
  const int nn = n * n;

  double* Vxx = bf.V;
  double* Vzx = bf.V + nn;
  double* Vzz = bf.V + 2 * nn;
  double* vx1 = bf.V + 3 * nn;
  double* vz1 = vx1 + n;
  double* F = bf.IN;
  double* Qxx = F + n * Fw;
  double* Qux = Qxx + nn;
  double* Quu = Qux + m * n;
  double* qx1 = Quu + m * m;
  double* qu1 = qx1 + n;
  double* P = bf.PGY;
  double* G = P + m * ldw;
  double* Y = G + m * ldw;
  double* Muu = bf.MUU;
  double* Lm = Muu + m * m;
  double* tau = bf.MISC;
  double* rdiag = tau + m;
  double* red = rdiag + m;
  int* iflag = reinterpret_cast<int*>(red + 32);
  int* sflag = iflag + 1;
  // rank-revealing slow path scratch (repair launches only, plq_rank.cuh)
  const RankScratch rsc =
      rank_scratch(a.rank_scratch + (REPAIR ? (int64_t)blockIdx.x * a.rank_scratch_doubles : 0), n, m, ldw);
  // blocked-factorization scratch (plq_blocked.cuh): block inverses, per-warp
  // tiles, V T' of the QR panel
  double* binv = red + 34;
  double* wsc = binv + ((m + 7) / 8) * 64;
  double* vts = wsc + (NT / 32) * 64;
  // shared-memory home of Muu for the blocked Cholesky (large mode, m <= 64), 16-byte aligned
  // (every MISC sub-buffer has an even length, so this stays 16-byte aligned)
  double* muus = (a.lay.large && sweep_muu_in_smem(n, m)) ? vts + 16 * n + 64 : nullptr;
  auto csync = [] { __syncthreads(); };
  const bool blocked = m >= 16;
  double* VF = bf.VF;
  double* Z = bf.Z;
  double* H = bf.H;

  // ---- initial value function and constraint rows (endpoint.py:182-199, serial.py:46-48)
  for (int idx = tid; idx < 3 * nn + 2 * n; idx += nt) bf.V[idx] = 0.0;
  if (tid == 0) *sflag = 0;
  __syncthreads();
  if (serial && a.smooth_vf0) {
    // smoothing pass: TerminalCost(Vxx, vx1 + Vzx' z) of segment j+1 (parallel.py:598-606)
    const double* v = a.smooth_vf0 + (b * J + j + 1) * (int64_t)(3 * nn + 2 * n);
    const double* z = a.smooth_links + (b * (J - 1) + j + 1) * (int64_t)n;
    for (int idx = tid; idx < nn; idx += nt) {
      const int i = idx / n, c = idx % n;
      Vxx[idx] = 0.5 * (v[i * n + c] + v[c * n + i]);
    }
    for (int i = tid; i < n; i += nt) {
      double t = 0.0;
      if (j + 1 < J - 1)
        for (int k = 0; k < n; ++k) t += v[nn + k * n + i] * z[k];
      vx1[i] = v[3 * nn + i] + t;
    }
  } else if (serial) {
    for (int idx = tid; idx < nn; idx += nt) Vxx[idx] = p.QxxT[b * nn + idx];
    for (int i = tid; i < n; i += nt) vx1[i] = p.qx1T[b * n + i];
  } else {
    for (int idx = tid; idx < n * ldw; idx += nt) {
      const int i = idx / ldw, c = idx % ldw;
      H[idx] = (c == i) ? 1.0 : ((c == n + i) ? -1.0 : 0.0);
    }
    if (a.endpoint_terminal && j == J - 1) {   // terminal cost + terminal rows (endpoint.py:178-191)
      for (int idx = tid; idx < nn; idx += nt) {
        const int i = idx / n, c = idx % n;
        Vxx[idx] = 0.5 * (p.QxxT[b * nn + i * n + c] + p.QxxT[b * nn + c * n + i]);
      }
      for (int i = tid; i < n; i += nt) vx1[i] = p.qx1T[b * n + i];
    }
  }
  int r = serial ? 0 : n;
  // collect_diagnostics: worst defects over the constrained stages (thread-uniform),
  // largest constraint-to-go row count (endpoint.py:200, 298-299)
  double defects[2] = {0.0, 0.0};
  int max_rows = r;
  if constexpr (!REPAIR) {
    if (a.force_repair && !serial) {
      // every endpoint segment goes to the rank-revealing launch (it has the singular vectors)
      if (tid == 0) {
        a.status[b * J + j] = PLQ_STATUS_RANK_REPAIR;
        push_repair(a, b, j);
      }
      __syncthreads();
      return;
    }
  }
  __syncthreads();

#ifdef PLQ_PHASE_PROFILE
  long long t_last = clock64();
#endif
  for (int s = L - 1; s >= 0; --s) {
    const int64_t st = b * T + (lo + s);
    // ---- stage inputs -> shared/scratch (coalesced global reads)
    // (streaming loads: read once, so they do not evict the L2-resident scratch)
    // Large mode: the Q blocks are not copied -- GEMM2 reads them from the
    // input arrays as addends loaded before its k-loop (less L2 scratch).
    const bool qdirect = bf.tiles != nullptr;
    const double* Qxx_s = qdirect ? p.Qxx + st * nn : Qxx;
    const double* Qux_s = qdirect ? p.Qux + st * m * n : Qux;
    const double* Quu_s = qdirect ? p.Quu + st * m * m : Quu;
    const double* qx1_s = qdirect ? p.qx1 + st * n : qx1;
    const double* qu1_s = qdirect ? p.qu1 + st * m : qu1;
    // Large mode: F = [Fx | Fu | f1] is not copied either -- the GEMMs take
    // Fx and Fu straight from the inputs (two operands instead of one)
    const double* fxp = qdirect ? p.Fx + st * nn : F;
    const double* fup = qdirect ? p.Fu + st * n * m : F + n;
    const double* f1p = qdirect ? p.f1 + st * n : nullptr;
    const int ldfx = qdirect ? n : Fw, ldfu = qdirect ? m : Fw;
    auto f1at = [&](int k) { return qdirect ? f1p[k] : F[k * Fw + n + m]; };
    auto fat = [&](int k, int c) { return c < n ? fxp[k * ldfx + c] : fup[k * ldfu + (c - n)]; };
    if (!qdirect) {
      for (int idx = tid; idx < nn; idx += nt) {
        F[(idx / n) * Fw + idx % n] = __ldcs(p.Fx + st * nn + idx);
        Qxx[idx] = __ldcs(p.Qxx + st * nn + idx);
      }
      for (int idx = tid; idx < n * m; idx += nt) {
        F[(idx / m) * Fw + n + idx % m] = __ldcs(p.Fu + st * n * m + idx);
        Qux[idx] = __ldcs(p.Qux + st * m * n + idx);
      }
      for (int i = tid; i < n; i += nt) {
        F[i * Fw + n + m] = __ldcs(p.f1 + st * n + i);
        qx1[i] = __ldcs(p.qx1 + st * n + i);
      }
      for (int idx = tid; idx < m * m; idx += nt) Quu[idx] = __ldcs(p.Quu + st * m * m + idx);
      for (int i = tid; i < m; i += nt) qu1[i] = __ldcs(p.qu1 + st * m + i);
    }
    __syncthreads();

    PLQ_GPH(0);
    // First stage of an endpoint segment: V = 0, [vx1; vz1] = 0 and the rows are
    // H = [I | -I | 0] (endpoint.py:182-191), so every product with V is an
    // exact zero and N = Hx F = F: the GEMMs of this stage reduce to copies.
    const bool vzero = a.lay.large && s == L - 1 && !serial && !(a.endpoint_terminal && j == J - 1);
    if (vzero) {
      for (int idx = tid; idx < n * Fw; idx += nt) {
        VF[idx] = 0.0;
        Z[idx] = 0.0;
      }
      for (int idx = tid; idx < m * nz; idx += nt) P[(idx / nz) * ldw + n + idx % nz] = 0.0;
    } else {
      // ---- GEMM1: [VF; Z] = [Vxx; Vzx] F  (endpoint.py:206-208, 212-213, 217).
      // The f1 column ([w; mz1] = [Vxx; Vzx] f1 + [vx1; vz1]) is a thread-per-row
      // matvec, so the GEMM's N is n + m (a whole 64-wide tile less in large mode)
      gemm_x<false, NT>(n + nz, n, n, bf.V, n, fxp, ldfx, bf.tiles, [&](int i, int c, double acc) {
        if (i < n) {
          VF[i * Fw + c] = acc;
        } else {
          Z[(i - n) * Fw + c] = acc;
        }
      });
      // (Mzu = Vzx Fu feeds only P's z-block, as Mzu': stored there directly)
      gemm_x<false, NT>(n + nz, m, n, bf.V, n, fup, ldfu, bf.tiles, [&](int i, int c, double acc) {
        if (i < n) {
          VF[i * Fw + n + c] = acc;
        } else {
          P[c * ldw + n + (i - n)] = acc;
        }
      });
      if (qdirect) {
        // warp per row, lanes over k: coalesced reads of V's rows (the scratch is in L2 / DRAM)
        const int lane = tid & 31, wp = tid >> 5, nwp = nt >> 5;
        for (int i0 = wp; i0 < n + nz; i0 += 2 * nwp) {
          const int i1 = i0 + nwp;
          const double* v0 = bf.V + (size_t)i0 * n;
          const double* v1 = bf.V + (size_t)(i1 < n + nz ? i1 : i0) * n;
          double t0 = 0.0, t1 = 0.0;
          for (int k = lane; k < n; k += 32) {
            const double f = f1p[k];
            t0 += v0[k] * f;
            t1 += v1[k] * f;
          }
          t0 = warp_sum(t0);
          t1 = warp_sum(t1);
          if (lane == 0) {
            if (i0 < n)
              VF[i0 * Fw + n + m] = vx1[i0] + t0;
            else
              Z[(i0 - n) * Fw + n + m] = vz1[i0 - n] + t0;
            if (i1 < n + nz) {
              if (i1 < n)
                VF[i1 * Fw + n + m] = vx1[i1] + t1;
              else
                Z[(i1 - n) * Fw + n + m] = vz1[i1 - n] + t1;
            }
          }
        }
      } else {
        for (int i = tid; i < n + nz; i += nt) {
          const double* vr = bf.V + (size_t)i * n;
          double t0 = 0.0, t1 = 0.0;
          int k = 0;
          for (; k + 1 < n; k += 2) {
            t0 += vr[k] * f1at(k);
            t1 += vr[k + 1] * f1at(k + 1);
          }
          if (k < n) t0 += vr[k] * f1at(k);
          if (i < n)
            VF[i * Fw + n + m] = vx1[i] + (t0 + t1);
          else
            Z[(i - n) * Fw + n + m] = vz1[i - n] + (t0 + t1);
        }
      }
    
    }
    __syncthreads();
    PLQ_GPH(1);
    if (vzero) {
      // M-terms with V = 0: the stage's own Q blocks (Mxx mirrored like the GEMM epilogue does)
      for (int i = tid; i < n + m; i += nt) {
        if (i < n)
          vx1[i] = qx1_s[i];
        else
          P[(i - n) * ldw + cc] = qu1_s[i - n];
      }
      for (int idx = tid; idx < nn; idx += nt) {
        const int i = idx / n, c = idx % n;
        if (c <= i) {
          const double v = __ldcs(Qxx_s + idx);
          Vxx[i * n + c] = v;
          Vxx[c * n + i] = v;
        }
      }
      for (int idx = tid; idx < m * n; idx += nt) P[(idx / n) * ldw + idx % n] = __ldcs(Qux_s + idx);
      for (int idx = tid; idx < m * m; idx += nt) Muu[idx] = __ldcs(Quu_s + idx);
    } else {
      // ---- GEMM2: M-terms (endpoint.py:209-211, 215-216); the w column
      // (mx1 = qx1 + Fx' w, mu1 = qu1 + Fu' w) again as a matvec
      for (int i = tid; i < n + m; i += nt) {
        double t0 = 0.0, t1 = 0.0;
        int k = 0;
        for (; k + 1 < n; k += 2) {
          t0 += fat(k, i) * VF[k * Fw + n + m];
          t1 += fat(k + 1, i) * VF[(k + 1) * Fw + n + m];
        }
        if (k < n) t0 += fat(k, i) * VF[k * Fw + n + m];
        if (i < n)
          vx1[i] = qx1_s[i] + (t0 + t1);   // mx1 in place (vx1 was consumed by GEMM1's f1 column)
        else
          P[(i - n) * ldw + cc] = qu1_s[i - n] + (t0 + t1);
      }
      // x rows over the x columns only (the Mxu block is never used), u rows
      // over all columns
      if (!gemm_x_pre_sym<true, NT>(
              n, n, fxp, ldfx, VF, Fw, bf.tiles, [&](int i, int c) { return c <= i ? __ldcs(Qxx_s + i * n + c) : 0.0; },
              [&](int i, int c, double v) {
                if (c <= i) {
                  Vxx[i * n + c] = v;
                  Vxx[c * n + i] = v;
                }
              }))
        gemm_x_pre<true, NT>(
            n, n, n, fxp, ldfx, VF, Fw, bf.tiles, [&](int i, int c) { return Qxx_s[i * n + c]; },
            [&](int i, int c, double v) { Vxx[i * n + c] = v; });   // Mxx in place (Vxx was consumed by GEMM1)
      gemm_x_pre<true, NT>(
          m, n + m, n, fup, ldfu, VF, Fw, bf.tiles,
          // (Q blocks are read once: streaming loads keep them from evicting the L2-resident scratch)
          [&](int u, int c) { return qdirect ? (c < n ? __ldcs(Qux_s + u * n + c) : __ldcs(Quu_s + u * m + (c - n)))
                                             : (c < n ? Qux_s[u * n + c] : Quu_s[u * m + (c - n)]); },
          [&](int u, int c, double v) {
            if (c < n)
              P[u * ldw + c] = v;
            else
              Muu[u * m + (c - n)] = v;
          });
    
    }
    __syncthreads();

    PLQ_GPH(2);
    // ---- gains
    bool chol = (r == 0);
    if (r != 0) {
      // constrained tail stage (endpoint.py:219-238, 251-252, 267-281)
      double part_h = 0.0, part_u = 0.0;
      for (int idx = tid; idx < r * n; idx += nt) {
        const double v = H[(idx / n) * ldw + idx % n];
        part_h += v * v;
      }
      for (int idx = tid; idx < n * m; idx += nt) {
        const double v = fup[(idx / m) * ldfu + idx % m];
        part_u += v * v;
      }
      const double hx2 = block_sum(part_h, red);
      const double fu2 = block_sum(part_u, red);
      const double nu_scale = sqrt(hx2) * sqrt(fu2);
      // N = Hx F -> VF (r x Fw): [Nx | Nu | Hx f1]
      if (vzero) {   // Hx = I
        for (int idx = tid; idx < nn; idx += nt) VF[(idx / n) * Fw + idx % n] = fxp[(idx / n) * ldfx + idx % n];
        for (int idx = tid; idx < n * m; idx += nt) VF[(idx / m) * Fw + n + idx % m] = fup[(idx / m) * ldfu + idx % m];
        for (int i = tid; i < n; i += nt) VF[i * Fw + n + m] = f1at(i);
      } else {
        gemm_x<false, NT>(r, n, n, H, ldw, fxp, ldfx, bf.tiles, [&](int i, int c, double acc) { VF[i * Fw + c] = acc; });
        gemm_x<false, NT>(r, m, n, H, ldw, fup, ldfu, bf.tiles,
                          [&](int i, int c, double acc) { VF[i * Fw + n + c] = acc; });
        for (int i = tid; i < r; i += nt) {
          double t = 0.0;
          for (int k = 0; k < n; ++k) t += H[i * ldw + k] * f1at(k);
          VF[i * Fw + n + m] = t;
        }
      }
      __syncthreads();
      PLQ_GPH(9);
      // stack [Nx | Nz=Hz | n1 = Hx f1 + h1] in place in H
      for (int idx = tid; idx < r * n; idx += nt) {
        const int i = idx / n, c = idx % n;
        H[i * ldw + c] = VF[i * Fw + c];
      }
      for (int i = tid; i < r; i += nt) H[i * ldw + cc] += VF[i * Fw + n + m];
      __syncthreads();
      PLQ_GPH(10);
      if (r >= m) {
        if (blocked && NT >= 256 && r <= 128)
          gqr8<NT / 32, decltype(csync), 4>(VF + n, r, m, Fw, H, W, ldw, rdiag, vts, wsc, tid, csync, vts + 8 * n,
                                            vts + 8 * n + 64);
        else if (blocked)
          gqr8<NT / 32>(VF + n, r, m, Fw, H, W, ldw, rdiag, vts, wsc, tid, csync);
        else
          cta_householder_qr(VF + n, r, m, Fw, H, W, ldw, tau, rdiag, red);
        PLQ_GPH(11);
        double rmax = 0.0, pf = 0.0;
        for (int i = 0; i < m; ++i) rmax = fmax(rmax, fabs(rdiag[i]));
        for (int idx = tid; idx < m * m; idx += nt) {
          const int i = idx / m, c = idx % m;
          const double v = c > i ? VF[i * Fw + n + c] : (c == i ? rdiag[i] : 0.0);
          pf += v * v;
        }
        const double thr = p.rank_tol * fmax(nu_scale, rmax);
        const double rf2 = block_sum(pf, red);
        if constexpr (REPAIR) {
          // rank-revealing path (plq_rank.cuh): SVD of R decides p exactly as
          // the reference does; gains, surviving rows, r - p rows left
          const double* Rv = VF + n;
          const int pr = rank_tail_solve(
              m, m, r, W, ldw, [&](int i, int c) { return c > i ? Rv[i * Fw + c] : (c == i ? rdiag[i] : 0.0); }, H, P,
              Muu, m, nu_scale, p.rank_tol, G, rsc, red, a.diag ? defects : nullptr);
          if (pr < 0) {
            if (tid == 0) *sflag = 1 + s;
            __syncthreads();
            break;
          }
          r -= pr;
          __syncthreads();
        } else {
        if (sqrt(rf2) <= thr) {
          // p = 0 for sure (sigma_max <= ||R||_F <= thr; Nu numerically zero,
          // e.g. a segment without control authority): the reflectors are
          // the identity, all r rows stay and the gains are the null-space
          // solve with Zw = I (endpoint.py:239-250)
          chol = true;
        } else {
          // G = -R^{-1} (Q1' stack): back substitution, thread per column
          // (blocked: in place on H's first m rows, DMMA tiles)
          if (blocked) {
            gtri_inv_upper8<NT / 32>(VF + n, m, Fw, rdiag, binv, tid, csync);
            gtrsm8<2, NT / 32, true>(VF + n, m, Fw, binv, H, W, ldw, wsc, tid, csync);
          }
          for (int c = tid; c < W && !blocked; c += nt) {
            for (int i = m - 1; i >= 0; --i) {
              double v = H[i * ldw + c];
              for (int k = i + 1; k < m; ++k) v -= VF[i * Fw + n + k] * G[k * ldw + c];
              G[i * ldw + c] = v / rdiag[i];
            }
          }
          __syncthreads();
          PLQ_GPH(12);
          double pz = 0.0;
          for (int idx = tid; idx < m * W; idx += nt) {
            const int u = idx / W, c = idx % W;
            const double g = -(blocked ? H[u * ldw + c] : G[u * ldw + c]);
            G[u * ldw + c] = g;
            if (c >= n && c < 2 * n) pz += g * g;
          }
          // p = m for sure iff sigma_min >= 1 / ||R^{-1}||_F = 1 / ||Kz||_F > thr
          // (plq_rank.cuh); otherwise the rank-revealing repair pass re-solves
          // this segment (NaN / Inf from an exactly singular R fail the test)
          const double kz2 = block_sum(pz, red);
          if (!(kz2 * thr * thr < 1.0)) {
            if (tid == 0) *sflag = PLQ_STATUS_RANK_REPAIR;
            __syncthreads();
            break;
          }
          // surviving rows Q2' stack: shift rows m..r-1 up by m, one block of
          // m rows at a time so sources and destinations never overlap
          for (int blk = 0; blk < r - m; blk += m) {
            const int rows = min(m, r - m - blk);
            for (int idx = tid; idx < rows * W; idx += nt) {
              const int i = blk + idx / W, c = idx % W;
              H[i * ldw + c] = H[(i + m) * ldw + c];
            }
            __syncthreads();
          }
          r -= m;
          __syncthreads();
        }
        }
      } else if (REPAIR) {
        // r < m, rank-revealing: QR of Nu' = Qw [Rw; 0], SVD of Rw' in the
        // Qw-rotated control coordinates (plq_rank.cuh), G = Qw G'
        double* X = rsc.wX;   // (the WIDE buffer exists only when n % m != 0)
        double* Mp = rsc.wM;
        double* Pp = rsc.wP;
        for (int idx = tid; idx < m * r; idx += nt) {
          const int c = idx / r, i = idx % r;
          X[c * r + i] = VF[i * Fw + n + c];
        }
        __syncthreads();
        cta_householder_qr(X, m, r, r, nullptr, 0, 1, tau, rdiag, red);
        for (int idx = tid; idx < m * m; idx += nt) Mp[idx] = Muu[idx];
        for (int idx = tid; idx < m * W; idx += nt) Pp[(idx / W) * ldw + idx % W] = P[(idx / W) * ldw + idx % W];
        __syncthreads();
        cta_apply_q(X, m, r, r, tau, Mp, m, m, false);
        for (int idx = tid; idx < m * m; idx += nt) {
          const int i = idx / m, c = idx % m;
          if (i < c) {
            const double t = Mp[i * m + c];
            Mp[i * m + c] = Mp[c * m + i];
            Mp[c * m + i] = t;
          }
        }
        __syncthreads();
        cta_apply_q(X, m, r, r, tau, Mp, m, m, false);
        cta_apply_q(X, m, r, r, tau, Pp, W, ldw, false);
        const int pr = rank_tail_solve(
            r, m, r, W, ldw, [&](int i, int c) { return c < i ? X[c * r + i] : (c == i ? rdiag[i] : 0.0); }, H, Pp,
            Mp, m, nu_scale, p.rank_tol, G, rsc, red, a.diag ? defects : nullptr);
        if (pr < 0) {
          if (tid == 0) *sflag = 1 + s;
          __syncthreads();
          break;
        }
        cta_apply_q(X, m, r, r, tau, G, W, ldw, true);
        r -= pr;
      } else {
        const int wr = wide_branch(p, n, m, r, W, ldw, Fw, VF, H, P, G, Muu, bf.WIDE, tau, rdiag, red, iflag,
                                   nu_scale, sflag, s);
        if (wr < 0) break;
        if (wr == 2) {
          if (tid == 0) *sflag = PLQ_STATUS_RANK_REPAIR;
          __syncthreads();
          break;
        }
        if (wr == 1) {
          chol = true;   // p = 0: all rows stay
        } else {
          r = 0;
        }
      }
    }
    PLQ_GPH(3);
    if (chol) {
      // G = -Muu^{-1} P: unconstrained stage, or p = 0 in a constrained one
      // (endpoint.py:239-250 with Zw = I; serial.py:63-70)
      // blocked: Cholesky of Muu in place (dead after this in Cholesky-gain
      // stages, which take the short value update) with the forward solve
      // fused in, G <- L^{-1}(-P); then the backward solve gives G directly
      if (!blocked) {
        for (int idx = tid; idx < m * m; idx += nt) Lm[idx] = Muu[idx];
        for (int idx = tid; idx < m * W; idx += nt) {
          const int u = idx / W, c = idx % W;
          G[u * ldw + c] = P[u * ldw + c];
        }
      }
      double* Mc = Muu;   // the factorization's working copy
      int ldm = m;
      if (blocked && muus != nullptr) {
        ldm = m + 4;
        Mc = muus;
        for (int idx = tid; idx < m * m; idx += nt) Mc[(idx / m) * ldm + idx % m] = Muu[idx];
      }
      if (tid == 0) *iflag = 0;
      __syncthreads();
      if (!(blocked ? gchol8<NT / 32, true>(Mc, m, ldm, binv, iflag, tid, csync, nullptr, G, W, ldw, wsc, P, -1.0)
                    : cta_cholesky(Lm, m, m, iflag))) {
        if (tid == 0) *sflag = 1 + s;
        __syncthreads();
        break;
      }
      PLQ_GPH(4);
      if (blocked) {
        gtrsm8<1, NT / 32, true>(Mc, m, ldm, binv, G, W, ldw, wsc, tid, csync);
      } else {
        cho_solve_x(Lm, m, m, G, W, ldw);
        for (int idx = tid; idx < m * W; idx += nt) {
          const int u = idx / W, c = idx % W;
          G[u * ldw + c] = -G[u * ldw + c];
        }
        __syncthreads();
      }
    }

    PLQ_GPH(5);
    // ---- policy outputs (parallel.py:224-236 stacking)
    for (int idx0 = tid; idx0 < m * n; idx0 += 4 * nt) {
      // four elements per trip, loads first (G is in L2 scratch); streaming
      // stores: the policies are not read again by this kernel
      double gx[4], gz[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = idx0 + e * nt;
        const int u = idx / n, c = idx % n;
        gx[e] = idx < m * n ? G[u * ldw + c] : 0.0;
        gz[e] = (idx < m * n && !serial) ? G[u * ldw + n + c] : 0.0;   // serial segment: Kz = 0
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = idx0 + e * nt;
        if (idx < m * n) {
          __stcs(a.Kx + st * m * n + idx, gx[e]);
          __stcs(a.Kz + st * m * n + idx, gz[e]);
        }
      }
    }
    for (int u = tid; u < m; u += nt) a.k1[st * m + u] = G[u * ldw + cc];

    // ---- value update (endpoint.py:285-294; serial.py:75-77)
    // Constrained stages: Y = P + Muu G and V += [P; G]'[G; Y] (the
    // reference's terms).  Stages whose gains came from the Cholesky branch
    // have G = -Muu^{-1} P, so Y = 0 in exact arithmetic and the update is the
    // standard Riccati form V += P'G (K = m: half the update, no Y GEMM), as
    // in the specialized kernels.
    PLQ_GPH(6);
    const int KV = chol ? m : 2 * m;
    if (!chol) {
      gemm_x<false, NT>(m, W, m, Muu, m, G, ldw, bf.tiles,
                        [&](int i, int c, double acc) { Y[i * ldw + c] = P[i * ldw + c] + acc; });
      __syncthreads();
    }
    // x rows over the x columns only (no discarded Vxz block), z rows over
    // [x | z] columns, the constant column as a matvec
    PLQ_GPH(7);
    // (the addends -- Mxx in Vxx, Mzx in Z, Vzz -- are loaded before each
    // tile's k-loop: L2 / DRAM latency of the scratch hides behind the DMMAs)
    const bool vsym = gemm_x_pre_sym<true, NT>(
        n, KV, P, ldw, G, ldw, bf.tiles, [&](int i, int c) { return c <= i ? Vxx[i * n + c] : 0.0; },
        [&](int i, int c, double v) {
          if (c <= i) {
            Vxx[i * n + c] = v;
            Vxx[c * n + i] = v;
          }
        });
    if (!vsym)
      gemm_x_pre<true, NT>(
          n, n, KV, P, ldw, G, ldw, bf.tiles, [&](int i, int c) { return Vxx[i * n + c]; },
          [&](int i, int c, double v) { Vxx[i * n + c] = v; });
    if (nz)
      gemm_x_pre<true, NT>(
          nz, 2 * n, KV, P + n, ldw, G, ldw, bf.tiles,
          [&](int zi, int c) { return c < n ? Z[zi * Fw + c] : Vzz[zi * n + (c - n)]; },
          [&](int zi, int c, double v) {
            if (c < n)
              Vzx[zi * n + c] = v;
            else
              Vzz[zi * n + (c - n)] = v;
          });
    for (int i = tid; i < n + nz; i += nt) {
      double t0 = 0.0, t1 = 0.0;
      int k = 0;
      for (; k + 1 < KV; k += 2) {
        t0 += P[k * ldw + i] * G[k * ldw + cc];
        t1 += P[(k + 1) * ldw + i] * G[(k + 1) * ldw + cc];
      }
      if (k < KV) t0 += P[k * ldw + i] * G[k * ldw + cc];
      if (i < n)
        vx1[i] += (t0 + t1);
      else
        vz1[i - n] = Z[(i - n) * Fw + n + m] + (t0 + t1);
    }
    __syncthreads();
    PLQ_GPH(8);
    // symmetrize Vxx: 0.5 * (V + V') (large mode: mirrored in the epilogues above)
    for (int idx = tid; idx < nn && !vsym; idx += nt) {
      const int i = idx / n, c = idx % n;
      if (i < c) {
        const double v = 0.5 * (Vxx[i * n + c] + Vxx[c * n + i]);
        Vxx[i * n + c] = v;
        Vxx[c * n + i] = v;
      }
    }
    __syncthreads();
  }
  // Vzz is never a GEMM operand: symmetrizing it once per segment is the same
  // linear map as every stage, sym(sym(A) + X) = sym(A + X)
  if (!serial) {
    for (int idx = tid; idx < nn; idx += nt) {
      const int i = idx / n, c = idx % n;
      if (i < c) {
        const double w = 0.5 * (Vzz[i * n + c] + Vzz[c * n + i]);
        Vzz[i * n + c] = w;
        Vzz[c * n + i] = w;
      }
    }
    __syncthreads();
  }

  // ---- segment-start value blocks (parallel.py:230-237) and status
  const int vsz = 3 * nn + 2 * n;
  if (a.vf0) {
    double* dst = a.vf0 + (b * J + j) * (int64_t)vsz;
    for (int idx = tid; idx < vsz; idx += nt) dst[idx] = bf.V[idx];
  }
  if (!serial && r > 0 && *sflag == 0 && a.feas) {
    // feasibility rows [Hx | Hz | h1] left at the segment start (parallel.py:452-456)
    double* dst = a.feas + (b * J + j) * (int64_t)n * (2 * n + 1);
    for (int idx = tid; idx < r * (2 * n + 1); idx += nt) {
      const int i = idx / (2 * n + 1), c = idx % (2 * n + 1);
      dst[idx] = H[i * ldw + c];
    }
  }
  if (a.diag != nullptr && tid == 0) {
    a.diag[(b * J + j) * 2] = defects[0];
    a.diag[(b * J + j) * 2 + 1] = defects[1];
    a.diag_rows[b * J + j] = max_rows;
  }
  if (tid == 0) {
    int st = *sflag;
    if (a.feas_rows) a.feas_rows[b * J + j] = (!serial && st == 0) ? r : 0;
    if (st == 0 && !serial && r > 0 && !a.feas) st = PLQ_STATUS_DEGENERATE;   // feasibility rows left
    a.status[b * J + j] = st;
    if (st == PLQ_STATUS_RANK_REPAIR) push_repair(a, b, j);
  }
  __syncthreads();
}

template <int NT, bool REPAIR>
__global__ void __launch_bounds__(NT, (NT == 256 ? 2 : 1)) sweep_kernel(SweepArgs a) {
  extern __shared__ __align__(16) double smem[];
  Bufs bf;
  double* ptrs[SB_COUNT];
  double* g = a.gscratch + (int64_t)blockIdx.x * a.lay.gmem_doubles;
#pragma unroll
  for (int i = 0; i < SB_COUNT; ++i) ptrs[i] = a.lay.in_smem[i] ? smem + a.lay.off[i] : g + a.lay.off[i];
  bf.V = ptrs[SB_V];
  bf.IN = ptrs[SB_IN];
  bf.PGY = ptrs[SB_PGY];
  bf.MUU = ptrs[SB_MUU];
  bf.MISC = ptrs[SB_MISC];
  bf.VF = ptrs[SB_VF];
  bf.Z = ptrs[SB_Z];
  bf.MX = ptrs[SB_MX];
  bf.H = ptrs[SB_H];
  bf.WIDE = ptrs[SB_WIDE];
  bf.tiles = a.lay.large ? smem + a.lay.tiles_off : nullptr;
  if constexpr (REPAIR) {
    // re-solve the segments the fast sweep could not decide (PLQ_STATUS_RANK_REPAIR)
    const long long flagged = (long long)*a.repair_ctr;
    for (long long i = blockIdx.x; i < flagged; i += gridDim.x) {
      const long long bj = a.repair_list[i];
      sweep_segment<NT, true>(a, bf, bj / a.p.J, (int)(bj % a.p.J));
    }
    return;
  }
  const int nloc = a.seg_end - a.seg_begin;
  const int64_t total = a.p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = a.seg_begin + (int)(task % nloc);
    if (!segment_bounds_ok(a.p, j)) {
      if (threadIdx.x == 0) a.status[b * a.p.J + j] = PLQ_STATUS_BAD_PARTITION;
      continue;
    }
    sweep_segment<NT, false>(a, bf, b, j);
  }
}

}  // namespace

// Launch / occupancy wrappers of one CTA size; each instantiation is compiled
// in its own translation unit (plq_sweep_t<NT>.cu) so the build parallelizes.
#ifdef PLQ_PHASE_PROFILE
#define PLQ_SWEEP_PHASE_ACCESSOR(NT)                                                                 \
  int sweep_phase_cycles_##NT(unsigned long long* out) {                                             \
    if (cudaMemcpyFromSymbol(out, g_gen_phase, sizeof(g_gen_phase)) != cudaSuccess) return -1;       \
    static unsigned long long zero[1024][16];                                                        \
    return cudaMemcpyToSymbol(g_gen_phase, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;              \
  }
#else
#define PLQ_SWEEP_PHASE_ACCESSOR(NT)
#endif

#define PLQ_SWEEP_INSTANTIATE(NT)                                                          \
  PLQ_SWEEP_PHASE_ACCESSOR(NT)                                                             \
  int launch_sweep_##NT(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) {       \
    sweep_kernel<NT, false><<<grid, NT, smem, s>>>(a);                                     \
    return cudaGetLastError() == cudaSuccess ? 0 : -1;                                     \
  }                                                                                        \
  int sweep_occupancy_##NT(size_t smem) {                                                  \
    int nb = 0;                                                                            \
    cudaFuncSetAttribute(sweep_kernel<NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)smem);                                                       \
    cudaFuncSetAttribute(sweep_kernel<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)smem);                                                       \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sweep_kernel<NT, false>, NT, smem); \
    return nb;                                                                             \
  }                                                                                        \
  int launch_sweep_repair_##NT(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) { \
    sweep_kernel<NT, true><<<grid, NT, smem, s>>>(a);                                      \
    return cudaGetLastError() == cudaSuccess ? 0 : -1;                                     \
  }

}  // namespace plq
