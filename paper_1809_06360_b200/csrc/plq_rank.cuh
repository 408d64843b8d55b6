// Rank-revealing constrained tail stage: the reference's SVD branch
// (endpoint.py:219-256) for the cases the fast kernels cannot decide.
//
// The fast paths factor Nu = Hx Fu by an unpivoted Householder QR and decide
// its rank p from two certificates that need no SVD:
//   * p = 0 for sure when  sigma_max(Nu) <= ||R||_F <= thr,
//   * p = m for sure when  sigma_min(Nu) >= 1 / ||R^{-1}||_F > thr,
// with thr = rank_tol * max(||Hx||_F ||Fu||_F, sigma_max) the reference's
// threshold (endpoint.py:226-231; ||Hx||_F ||Fu||_F >= ||Nu||_F >= sigma_max,
// so it equals rank_tol * ||Hx||_F ||Fu||_F).  ||R^{-1}||_F comes for free:
// the z-block of the gains is Kz = -R^{-1} Q1' Hz and the rows of Hz stay
// orthonormal through every tail stage (Hz starts at -I and is only ever
// rotated / row-selected), so ||Kz||_F = ||R^{-1}||_F.  A stage that meets
// neither certificate (sigma_min within a factor sqrt(m) of the threshold,
// or 0 < p < m) is re-solved here from the singular values, exactly as the
// reference decides: p = #{sigma_i > thr}.
//
// Everything is expressed in "primed" coordinates in which Nu has the
// k x k block S in its top-left corner (k = min(r, m)):
//   r >= m:  Nu = Q [R; 0]      -> S = R,   rows rotated by Q (H = Q' stack)
//   r <  m:  Nu = [Rw' 0] Qw'   -> S = Rw', controls rotated by Qw
// With S = U diag(sigma) V' (one-sided Jacobi):
//   base' = [V_p sigma_p^{-1} U_p' stack'_{0:k}; 0]                 (:234-238)
//   Zw'   = [[V_{p:}, 0], [0, I_{m-k}]]                             (:239-241)
//   G'    = -(base' + Zw' (Zw' Muu' Zw')^{-1} Zw' (P' - Muu' base')) (:242-250)
//   rows' = [U_perp' stack'_{0:k}; stack'_{k:r}]   (r - p rows; the projector
//           I - U_p U_p' of :267-270 followed by the compression of
//           :271-281, whose [Hx Hz] rows keep full row rank because their
//           Hz block is orthonormal)
// U_perp is completed by a Householder QR of U_p (an exactly orthonormal
// basis of the complement).
#pragma once

#include "plq_device.cuh"

namespace plq {

// doubles of per-CTA scratch the slow path needs for state dim n, control
// dim m, row width W (leading dimension ldw >= W)
__host__ __device__ inline size_t rank_scratch_doubles(int n, int m, int ldw) {
  const size_t k = (size_t)(n < m ? n : m);
  const size_t mm = (size_t)m;
  return 3 * k * k + 4 * k + 4 * mm * (size_t)ldw + 5 * mm * mm + 3 * mm + 64;
}

struct RankScratch {
  double *A, *V, *sig, *UP, *base, *C, *Wm, *Zw, *T1, *tau, *rd;
  double *wX, *wM, *wP;   // r < m caller: Nu' QR factors, Qw' Muu Qw, Qw' P
  int* perm;
  int* flag;
};

__device__ inline RankScratch rank_scratch(double* s, int n, int m, int ldw) {
  const int k = n < m ? n : m;
  RankScratch r;
  r.A = s;
  r.V = r.A + k * k;
  r.UP = r.V + k * k;
  r.sig = r.UP + k * k;
  r.base = r.sig + k;
  r.C = r.base + m * ldw;
  r.Wm = r.C + m * ldw;
  r.Zw = r.Wm + m * m;
  r.T1 = r.Zw + m * m;
  r.tau = r.T1 + m * m + m * ldw;   // T1 doubles as the q x W solve block
  r.rd = r.tau + m + k;
  r.wX = r.rd + m + k;
  r.wM = r.wX + m * m;
  r.wP = r.wM + m * m;
  r.perm = reinterpret_cast<int*>(r.wP + m * ldw);
  r.flag = r.perm + k + 1;
  return r;
}

// One-sided (Hestenes) Jacobi SVD of the k x k matrix held column-major in
// A (A[c*k + i]).  On exit the columns of A are sigma_j u_j, V (column-major)
// holds the right singular vectors, sig the sigma_j and perm the column
// order by decreasing sigma.  Pairs of a round-robin tournament round are
// disjoint, so each warp rotates its pairs independently.
__device__ inline void cta_jacobi_svd(double* A, double* V, double* sig, int* perm, int k, int* flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) V[idx] = (idx / k == idx % k) ? 1.0 : 0.0;
  const int K = k + (k & 1);
  __syncthreads();
  for (int sweep = 0; sweep < 60 && K > 1; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int t = 0; t < K - 1; ++t) {
      for (int pi = warp; pi < K / 2; pi += nw) {
        const int a = pi == 0 ? 0 : 1 + ((pi - 1 + t) % (K - 1));
        const int b = 1 + ((K - 2 - pi + t) % (K - 1));
        if (a >= k || b >= k) continue;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < k; i += 32) {
          const double x = A[a * k + i], y = A[b * k + i];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
        for (int i = lane; i < k; i += 32) {
          const double x = A[a * k + i], y = A[b * k + i];
          A[a * k + i] = c * x - s * y;
          A[b * k + i] = s * x + c * y;
          const double vx = V[a * k + i], vy = V[b * k + i];
          V[a * k + i] = c * vx - s * vy;
          V[b * k + i] = s * vx + c * vy;
        }
        if (lane == 0) *flag = 1;
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  for (int j = warp; j < k; j += nw) {
    double s2 = 0.0;
    for (int i = lane; i < k; i += 32) s2 += A[j * k + i] * A[j * k + i];
    s2 = warp_sum(s2);
    if (lane == 0) sig[j] = sqrt(s2);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < k; ++j) perm[j] = j;
    for (int j = 0; j < k; ++j) {   // selection sort, descending (k <= 128)
      int best = j;
      for (int i = j + 1; i < k; ++i)
        if (sig[perm[i]] > sig[perm[best]]) best = i;
      const int tmp = perm[j];
      perm[j] = perm[best];
      perm[best] = tmp;
    }
  }
  __syncthreads();
}

// The slow path in primed coordinates (see the file comment).  S(i, c) is
// read through `sat`; H holds stack' (r rows, stride ldw, W columns), Pp the
// m x W block [Mux | Mzu' | mu1]' (stride ldw), Mp = Muu' (stride ldm).
// Writes G' (stride ldw) and the surviving rows into H[0 : r - p]; returns p,
// or -1 when W = Zw' Muu' Zw' is not positive definite (CholeskyFailure).
template <class SAt>
__device__ int rank_tail_solve(int k, int m, int r, int W, int ldw, SAt sat, double* H, const double* Pp,
                               const double* Mp, int ldm, double nu_scale, double rank_tol, double* G,
                               const RankScratch& s, double* red, double* defects = nullptr) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int idx = tid; idx < k * k; idx += nt) {
    const int c = idx / k, i = idx % k;
    s.A[idx] = sat(i, c);   // column-major
  }
  __syncthreads();
  cta_jacobi_svd(s.A, s.V, s.sig, s.perm, k, s.flag);
  const double smax = k > 0 ? s.sig[s.perm[0]] : 0.0;
  const double thr = rank_tol * fmax(nu_scale, smax);
  int p = 0;
  for (int j = 0; j < k; ++j) p += s.sig[s.perm[j]] > thr ? 1 : 0;
  // U_p (k x p, stride k) and Y = sigma_p^{-1} U_p' stack'_{0:k} (p x W in C)
  for (int idx = tid; idx < k * p; idx += nt) {
    const int i = idx / p, c = idx % p;
    const int col = s.perm[c];
    s.UP[i * k + c] = s.A[col * k + i] / s.sig[col];
  }
  __syncthreads();
  if (defects != nullptr) {
    // StageDiagnostics (endpoint.py:258-276), thread-uniform maxima:
    // basis: |V V' - I| of the k x k right singular basis ([Py | Zw] in these
    // coordinates; zero by definition when p = 0); projector: P = I - U_p U_p',
    // P P - P = U_p (U_p'U_p - I) U_p'
    double bd = 0.0, pd = 0.0;
    if (p > 0) {
      for (int idx = tid; idx < k * k; idx += nt) {
        const int i = idx / k, c = idx % k;
        double v = (i == c) ? -1.0 : 0.0;
        for (int l = 0; l < k; ++l) v += s.V[l * k + i] * s.V[l * k + c];
        bd = fmax(bd, fabs(v));
      }
      // E = U_p'U_p - I in T1 (p x p), then U_p E U_p'
      for (int idx = tid; idx < p * p; idx += nt) {
        const int a = idx / p, c = idx % p;
        double v = (a == c) ? -1.0 : 0.0;
        for (int i = 0; i < k; ++i) v += s.UP[i * k + a] * s.UP[i * k + c];
        s.T1[idx] = v;
      }
      __syncthreads();
      // F = E U_p' (p x k) in C (free until the next product), then U_p F
      for (int idx = tid; idx < p * k; idx += nt) {
        const int a = idx / k, c = idx % k;
        double t = 0.0;
        for (int e = 0; e < p; ++e) t += s.T1[a * p + e] * s.UP[c * k + e];
        s.C[idx] = t;
      }
      __syncthreads();
      for (int idx = tid; idx < k * k; idx += nt) {
        const int i = idx / k, c = idx % k;
        double v = 0.0;
        for (int a = 0; a < p; ++a) v += s.UP[i * k + a] * s.C[a * k + c];
        pd = fmax(pd, fabs(v));
      }
    }
    bd = block_max(bd, red);
    pd = block_max(pd, red);
    defects[0] = fmax(defects[0], bd);
    defects[1] = fmax(defects[1], pd);
    __syncthreads();
  }
  cta_gemm<true, false, 1, 1>(p, W, k, s.UP, k, H, ldw, [&](int c, int w, double acc) {
    s.C[c * ldw + w] = acc / s.sig[s.perm[c]];
  });
  __syncthreads();
  // base' = [V_p Y; 0]
  for (int idx = tid; idx < m * W; idx += nt) {
    const int i = idx / W, w = idx % W;
    double v = 0.0;
    if (i < k)
      for (int c = 0; c < p; ++c) v += s.V[s.perm[c] * k + i] * s.C[c * ldw + w];
    s.base[i * ldw + w] = v;
  }
  __syncthreads();
  if (p < m) {
    const int q = m - p;
    // Zw' (m x q, stride q)
    for (int idx = tid; idx < m * q; idx += nt) {
      const int i = idx / q, c = idx % q;
      double v;
      if (c < k - p)
        v = i < k ? s.V[s.perm[p + c] * k + i] : 0.0;
      else
        v = (i >= k && i - k == c - (k - p)) ? 1.0 : 0.0;
      s.Zw[idx] = v;
    }
    // C = P' - Muu' base'
    __syncthreads();
    cta_gemm<false, false, 1, 1>(m, W, m, Mp, ldm, s.base, ldw,
                                 [&](int i, int w, double acc) { s.C[i * ldw + w] = Pp[i * ldw + w] - acc; });
    cta_gemm<false, false, 1, 1>(m, q, m, Mp, ldm, s.Zw, q, [&](int i, int c, double acc) { s.T1[i * q + c] = acc; });
    __syncthreads();
    cta_gemm<true, false, 1, 1>(q, q, m, s.Zw, q, s.T1, q, [&](int i, int c, double acc) { s.Wm[i * q + c] = acc; });
    __syncthreads();
    if (!cta_cholesky(s.Wm, q, q, nullptr)) return -1;
    // X = Wm^{-1} Zw' C (q x W, in T1), G' = -(base' + Zw' X)
    cta_gemm<true, false, 1, 1>(q, W, m, s.Zw, q, s.C, ldw, [&](int i, int w, double acc) { s.T1[i * ldw + w] = acc; });
    __syncthreads();
    cta_cho_solve(s.Wm, q, q, s.T1, W, ldw);
    cta_gemm<false, false, 1, 1>(m, W, q, s.Zw, q, s.T1, ldw, [&](int i, int w, double acc) {
      G[i * ldw + w] = -(s.base[i * ldw + w] + acc);
    });
  } else {
    for (int idx = tid; idx < m * W; idx += nt) G[(idx / W) * ldw + idx % W] = -s.base[(idx / W) * ldw + idx % W];
  }
  __syncthreads();
  if (p > 0) {
    // rows: Q_c' stack'_{0:k} with Q_c = [U_p | U_perp] from a QR of U_p,
    // keep rows p..k-1, then stack'_{k:r}; shift up by p (row by row, the
    // destination always precedes the source)
    cta_householder_qr(s.UP, k, p, k, H, W, ldw, s.tau, s.rd, red);
    for (int i = 0; i < r - p; ++i) {
      for (int w = tid; w < W; w += nt) H[i * ldw + w] = H[(i + p) * ldw + w];
      __syncthreads();
    }
  }
  return p;
}

}  // namespace plq
