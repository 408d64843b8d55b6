// Two-point-boundary solve (endpoint.py:303-653): solve_endpoint_affine and
// EndpointAffineSolution.evaluate for a batch of problems.
//
//   K1 (sweep kernels, endpoint mode seeded with the terminal cost):
//       backward_pass(stages, terminal) -> Kx, Kz, k1, value at t = 0.
//   ep_maps_kernel:   forward_pass (:326-349) -- X_t = [Ra|Rz|r1] (n x W),
//       S_t = [Sa|Sz|s1] (m x W), W = 2n+1, stepped on the FP64 tensor pipe:
//       S_t = Kx X_t + [0|Kz|k1],  X_{t+1} = Fx X_t + Fu S_t + [0|0|f1].
//   ep_mult_kernel:   assemble_normal_equations + multiplier_pass
//       (:370-476) -- the (T+2)-block Gram system over lam_0..lam_T, mu with
//       the W-wide right-hand side, assembled block by block on the fly and
//       factored by block Cholesky (solve_block_tridiagonal, :410-438), then
//       back-substituted in place: Lam_t = [La|Lz|l1], E = [Ea|Ez|e1].
//   ep_point_kernel + ep_eval_kernel + ep_fin_kernel: evaluate (:538-575)
//       at (x_init, x_term): states / controls / lambdas / mu from the maps,
//       objective and the full KKT stack (problem.py:366-420), stage-parallel.
//
// The maps / multiplier recurrences are sequential in t (as in the
// reference): one CTA per problem, the batch gives the parallelism.  Their
// operands live in the output arrays and a per-problem slice of global
// scratch (L2-resident), read back within the kernel through coherent loads.
#include <cuda_runtime.h>

#include "plq_device.cuh"
#include "plq_internal.h"

namespace plq {
namespace {

constexpr int EP_NT = 256;
constexpr int EP_CH = 8;

// C(MxN) = op(A) op(B) through DMMA (cta_gemm without the read-only
// qualifiers: operands may have been written earlier by this CTA).
template <bool TA, bool TB, int BM, int BN, class Epi>
__device__ __forceinline__ void gemm_c(int M, int N, int K, const double* A, int lda, const double* B, int ldb,
                                       Epi epi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int tm_count = (M + 8 * BM - 1) / (8 * BM);
  const int tn_count = (N + 8 * BN - 1) / (8 * BN);
  for (int tile = warp; tile < tm_count * tn_count; tile += nwarps) {
    const int i0 = (tile / tn_count) * 8 * BM;
    const int j0 = (tile % tn_count) * 8 * BN;
    double acc[BM][BN][2];
#pragma unroll
    for (int a = 0; a < BM; ++a)
#pragma unroll
      for (int b = 0; b < BN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 2
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int kk = k0 + q;
      double av[BM], bv[BN];
#pragma unroll
      for (int a = 0; a < BM; ++a) {
        const int i = i0 + 8 * a + g;
        av[a] = (i < M && kk < K) ? (TA ? A[(size_t)kk * lda + i] : A[(size_t)i * lda + kk]) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < BN; ++b) {
        const int j = j0 + 8 * b + g;
        bv[b] = (j < N && kk < K) ? (TB ? B[(size_t)j * ldb + kk] : B[(size_t)kk * ldb + j]) : 0.0;
      }
#pragma unroll
      for (int a = 0; a < BM; ++a)
#pragma unroll
        for (int b = 0; b < BN; ++b) dmma884(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
#pragma unroll
    for (int a = 0; a < BM; ++a)
#pragma unroll
      for (int b = 0; b < BN; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = i0 + 8 * a + g, j = j0 + 8 * b + 2 * q + e;
          if (i < M && j < N) epi(i, j, acc[a][b][e]);
        }
  }
}

struct EpArgs {
  plq_problem_t p;
  plq_endpoint_outputs_t o;
  double* Xb;        // (B,T+1,n,n) block-Cholesky X_i
  double* scratch;   // (B, EP_SCRATCH) per-problem work blocks
  const double* x_init;
  const double* x_term;
  plq_endpoint_point_t pt;
  double* part;      // (B, nch, 2) objective / KKT partials
  int nch;
};

__host__ __device__ inline int64_t ep_scratch(int n, int m) {
  const int64_t W = 2 * n + 1;
  return 2 * n * W + m * W + 2LL * n * n;
}

// ---- forward_pass (endpoint.py:326-349)
template <int NT, bool ONCHIP>
__global__ void __launch_bounds__(NT) ep_maps_kernel(EpArgs a) {
  extern __shared__ __align__(16) double esm[];
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, W = 2 * n + 1, tid = threadIdx.x;
  const int64_t b = blockIdx.x, nn = (int64_t)n * n, nm = (int64_t)n * m;
  double* X0 = a.o.X + b * (T + 1) * n * W;
  // ONCHIP: X_t ping-pongs and S_t lives in shared memory (the GEMM operands),
  // each is streamed out to the output maps once
  double* XS[2] = {esm, esm + n * W};
  double* SS = esm + 2 * n * W;
  for (int idx = tid; idx < n * W; idx += NT) {
    const double v = (idx / W == idx % W) ? 1.0 : 0.0;
    X0[idx] = v;
    if (ONCHIP) XS[0][idx] = v;
  }
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    const int64_t bt = b * T + t;
    double* Xg = X0 + (int64_t)t * n * W;
    double* Sg = a.o.S + bt * m * W;
    double* X = ONCHIP ? XS[t & 1] : Xg;
    double* Xn = ONCHIP ? XS[(t + 1) & 1] : Xg + n * W;
    double* S = ONCHIP ? SS : Sg;
    const double* Kz = a.o.Kz + bt * nm;
    const double* k1 = a.o.k1 + bt * m;
    gemm_c<false, false, 1, 2>(m, W, n, a.o.Kx + bt * nm, n, X, W, [&](int i, int c, double v) {
      S[i * W + c] = v + (c >= n && c < 2 * n ? Kz[i * n + (c - n)] : (c == 2 * n ? k1[i] : 0.0));
    });
    __syncthreads();
    const double* f1 = p.f1 + bt * n;
    gemm_c<false, false, 1, 2>(n, W, n, p.Fx + bt * nn, n, X, W, [&](int i, int c, double v) {
      Xn[i * W + c] = v + (c == 2 * n ? f1[i] : 0.0);
    });
    __syncthreads();
    gemm_c<false, false, 1, 2>(n, W, m, p.Fu + bt * nm, m, S, W, [&](int i, int c, double v) { Xn[i * W + c] += v; });
    __syncthreads();
    if (ONCHIP) {
      for (int idx = tid; idx < m * W; idx += NT) Sg[idx] = S[idx];
      for (int idx = tid; idx < n * W; idx += NT) Xg[n * W + idx] = Xn[idx];
    }
  }
}

// bx(t) = -(Qxx_t X_t + Qux_t' S_t) - [0|0|qx1_t]  (t < T);  -(QxxT X_T) - [0|0|qx1T]
__device__ void ep_bx(const EpArgs& a, int64_t b, int t, double* BX) {
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, W = 2 * n + 1;
  const int64_t nn = (int64_t)n * n, nm = (int64_t)n * m;
  const double* X = a.o.X + (b * (T + 1) + t) * n * W;
  if (t < T) {
    const int64_t bt = b * T + t;
    const double* q = p.qx1 + bt * n;
    gemm_c<false, false, 1, 2>(n, W, n, p.Qxx + bt * nn, n, X, W, [&](int i, int c, double v) {
      BX[i * W + c] = -v - (c == 2 * n ? q[i] : 0.0);
    });
    __syncthreads();
    gemm_c<true, false, 1, 2>(n, W, m, p.Qux + bt * nm, n, a.o.S + bt * m * W, W,
                              [&](int i, int c, double v) { BX[i * W + c] -= v; });
  } else {
    const double* q = p.qx1T + b * n;
    gemm_c<false, false, 1, 2>(n, W, n, p.QxxT + b * nn, n, X, W, [&](int i, int c, double v) {
      BX[i * W + c] = -v - (c == 2 * n ? q[i] : 0.0);
    });
  }
  __syncthreads();
}

// bu(t) = -(Qux_t X_t + Quu_t S_t) - [0|0|qu1_t]
__device__ void ep_bu(const EpArgs& a, int64_t b, int t, double* BU) {
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, W = 2 * n + 1;
  const int64_t bt = b * T + t, nm = (int64_t)n * m;
  const double* q = p.qu1 + bt * m;
  gemm_c<false, false, 1, 2>(m, W, n, p.Qux + bt * nm, n, a.o.X + (b * (T + 1) + t) * n * W, W,
                             [&](int i, int c, double v) { BU[i * W + c] = -v - (c == 2 * n ? q[i] : 0.0); });
  __syncthreads();
  gemm_c<false, false, 1, 2>(m, W, m, p.Quu + bt * (int64_t)m * m, m, a.o.S + bt * m * W, W,
                             [&](int i, int c, double v) { BU[i * W + c] -= v; });
  __syncthreads();
}

// ---- assemble_normal_equations + multiplier_pass (endpoint.py:370-476)
template <int EP_NT, bool ONCHIP>
__global__ void __launch_bounds__(EP_NT) ep_mult_kernel(EpArgs a) {
  __shared__ int flag;
  extern __shared__ __align__(16) double esm[];
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, W = 2 * n + 1, tid = threadIdx.x;
  const int64_t b = blockIdx.x, nn = (int64_t)n * n, nm = (int64_t)n * m;
  // ONCHIP: the work blocks, d_i and X_i (ping-pong) in shared memory; d_i
  // and X_i are streamed out once for the back substitution
  double* sc = ONCHIP ? esm : a.scratch + b * ep_scratch(n, m);
  double* BX = sc;             // bx[t]       n x W
  double* BXn = BX + n * W;    // bx[t+1]     n x W
  double* BU = BXn + n * W;    // bu[t]       m x W
  double* P = BU + m * W;      // pivot block n x n (Cholesky in place)
  double* Y = P + nn;          // Fx' + X_{i-1}  n x n
  double* DB[2] = {Y + nn, Y + nn + n * W};
  double* XB[2] = {DB[1] + n * W, DB[1] + n * W + nn};
  double* Xb = a.Xb + b * (T + 1) * nn;
  double* Lam = a.o.Lam + b * (T + 1) * n * W;
  double* E = a.o.E + b * n * W;
  if (a.o.feas_rows != nullptr && a.o.feas_rows[b] > 0) {
    // unreachable endpoint rows: the boundary constraints are linearly
    // dependent, the Gram system is singular and the reference computes no
    // multiplier maps (endpoint.py:607-613); evaluate uses gradient duals
    if (tid == 0) a.o.gram_status[b] = -1;
    return;
  }
  int fail = 0;
  for (int i = 0; i <= T + 1 && !fail; ++i) {
    double* dg = (i <= T) ? Lam + (int64_t)i * n * W : E;   // d_i's home
    double* d = ONCHIP ? DB[i & 1] : dg;
    if (i == 0) {
      ep_bx(a, b, 0, BX);
      for (int idx = tid; idx < n * W; idx += EP_NT) d[idx] = BX[idx];
      for (int idx = tid; idx < n * n; idx += EP_NT) P[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
    } else if (i <= T) {
      const int t = i - 1;
      const int64_t bt = b * T + t;
      const double* Fx = p.Fx + bt * nn;
      const double* Fu = p.Fu + bt * nm;
      const double* dprev = ONCHIP ? DB[(i - 1) & 1] : Lam + (int64_t)(i - 1) * n * W;
      ep_bu(a, b, t, BU);
      ep_bx(a, b, t + 1, BXn);
      // g = bx[t+1] - Fx (bx[t] - d_{i-1}) - Fu bu[t]
      for (int idx = tid; idx < n * W; idx += EP_NT) BX[idx] -= dprev[idx];
      // P = I + Fx (Fx' + X_{i-1}) + Fu Fu'
      const double* Xprev = ONCHIP ? XB[(i - 1) & 1] : Xb + (int64_t)(i - 1) * nn;
      for (int idx = tid; idx < n * n; idx += EP_NT) {
        const int r = idx / n, c = idx % n;
        Y[idx] = Fx[c * n + r] + Xprev[idx];
      }
      __syncthreads();
      gemm_c<false, false, 1, 2>(n, W, n, Fx, n, BX, W, [&](int r, int c, double v) { d[r * W + c] = BXn[r * W + c] - v; });
      gemm_c<false, false, 1, 1>(n, n, n, Fx, n, Y, n, [&](int r, int c, double v) {
        P[r * n + c] = (r == c ? 1.0 : 0.0) + v;
      });
      __syncthreads();
      gemm_c<false, false, 1, 2>(n, W, m, Fu, m, BU, W, [&](int r, int c, double v) { d[r * W + c] -= v; });
      gemm_c<false, true, 1, 1>(n, n, m, Fu, m, Fu, m, [&](int r, int c, double v) { P[r * n + c] += v; });
      __syncthreads();
      double* tmp = BX;   // bx[t+1] becomes bx[t] of the next block
      BX = BXn;
      BXn = tmp;
    } else {
      // mu block: P = I - X_T, g = bx[T] - d_T
      const double* dprev = ONCHIP ? DB[T & 1] : Lam + (int64_t)T * n * W;
      const double* Xprev = ONCHIP ? XB[T & 1] : Xb + (int64_t)T * nn;
      for (int idx = tid; idx < n * W; idx += EP_NT) d[idx] = BX[idx] - dprev[idx];
      for (int idx = tid; idx < n * n; idx += EP_NT) P[idx] = (idx / n == idx % n ? 1.0 : 0.0) - Xprev[idx];
    }
    __syncthreads();
    if (!cta_cholesky(P, n, n, &flag)) {
      fail = 1 + i;
      break;
    }
    cta_cho_solve(P, n, n, d, W, W);
    if (ONCHIP)
      for (int idx = tid; idx < n * W; idx += EP_NT) dg[idx] = d[idx];
    if (i <= T) {
      // X_i = P^{-1} sub_i',  sub_i = -Fx_i (i < T), I (i = T)
      double* Xi = ONCHIP ? XB[i & 1] : Xb + (int64_t)i * nn;
      const double* Fxi = p.Fx + (b * T + i) * nn;
      for (int idx = tid; idx < n * n; idx += EP_NT) {
        const int r = idx / n, c = idx % n;
        Xi[idx] = (i < T) ? -Fxi[c * n + r] : (r == c ? 1.0 : 0.0);
      }
      __syncthreads();
      cta_cho_solve(P, n, n, Xi, n, n);
      if (ONCHIP)
        for (int idx = tid; idx < n * n; idx += EP_NT) Xb[(int64_t)i * nn + idx] = Xi[idx];
    }
    __syncthreads();
  }
  if (tid == 0) a.o.gram_status[b] = fail;
  if (fail) return;
  // back substitution: out_{T+1} = d_{T+1}; out_i = d_i - X_i out_{i+1}
  for (int i = T; i >= 0; --i) {
    double* di = Lam + (int64_t)i * n * W;
    const double* next = (i == T) ? E : di + n * W;
    gemm_c<false, false, 1, 2>(n, W, n, Xb + (int64_t)i * nn, n, next, W, [&](int r, int c, double v) { di[r * W + c] -= v; });
    __syncthreads();
  }
}

// ---- evaluate (endpoint.py:538-575): trajectories from the maps
__global__ void __launch_bounds__(EP_NT) ep_point_kernel(EpArgs a) {
  extern __shared__ double v[];   // [x_init; x_term; 1]
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, W = 2 * n + 1, tid = threadIdx.x;
  const int64_t b = blockIdx.x / a.nch;
  const int c = (int)(blockIdx.x % a.nch);
  // problems with feasibility rows have no multiplier maps: ep_dual_kernel fills lam / mu
  const bool dual = a.o.feas_rows != nullptr && a.o.feas_rows[b] > 0;
  for (int i = tid; i < W; i += EP_NT)
    v[i] = i < n ? a.x_init[b * n + i] : (i < 2 * n ? a.x_term[b * n + i - n] : 1.0);
  __syncthreads();
  const int t0 = c * EP_CH, t1 = min(T + 1, t0 + EP_CH);
  for (int t = t0; t < t1; ++t) {
    const double* X = a.o.X + (b * (T + 1) + t) * n * W;
    const double* L = a.o.Lam + (b * (T + 1) + t) * n * W;
    for (int r = tid; r < (dual ? n : 2 * n); r += EP_NT) {
      const double* row = (r < n ? X : L) + (r % n) * W;
      double s = 0.0;
      for (int k = 0; k < W; ++k) s += row[k] * v[k];
      (r < n ? a.pt.x : a.pt.lam)[(b * (T + 1) + t) * n + r % n] = s;
    }
    if (t < T) {
      const double* S = a.o.S + (b * T + t) * m * W;
      for (int r = tid; r < m; r += EP_NT) {
        double s = 0.0;
        for (int k = 0; k < W; ++k) s += S[r * W + k] * v[k];
        a.pt.u[(b * T + t) * m + r] = s;
      }
    } else if (!dual) {
      for (int r = tid; r < n; r += EP_NT) {
        double s = 0.0;
        for (int k = 0; k < W; ++k) s += a.o.E[(b * n + r) * W + k] * v[k];
        a.pt.mu[b * n + r] = s;
      }
    }
  }
}

// Problems with feasibility rows (unreachable endpoint directions): the
// residual of the rows at (x_init, x_term) (feasibility_residual,
// endpoint.py:507-511) and the multipliers from the value-function gradient
// and the stationarity recursion (gradient_duals, endpoint.py:566-587):
//   mu = -(Vzx0 x_init + Vzz0 x_term + vz10),  lam_T = -(QxxT x_T + qx1T) - mu,
//   lam_t = Fx_t' lam_{t+1} - (Qxx_t x_t + Qux_t' u_t + qx1_t).
// One CTA per problem (the recursion is sequential in t); no-op without rows.
__global__ void __launch_bounds__(EP_NT) ep_dual_kernel(EpArgs a) {
  extern __shared__ double dsm[];   // lam ping | lam pong | x_init | x_term
  __shared__ double red[32];
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, W = 2 * n + 1, tid = threadIdx.x;
  const int64_t b = blockIdx.x, nn = (int64_t)n * n, nm = (int64_t)n * m;
  const int rows = a.o.feas_rows != nullptr ? a.o.feas_rows[b] : 0;
  if (rows <= 0) {
    if (tid == 0 && a.pt.feas_residual != nullptr) a.pt.feas_residual[b] = 0.0;
    return;
  }
  double* l0 = dsm;
  double* l1 = dsm + n;
  double* xi = l1 + n;
  double* xt = xi + n;
  for (int i = tid; i < n; i += EP_NT) {
    xi[i] = a.x_init[b * n + i];
    xt[i] = a.x_term[b * n + i];
  }
  __syncthreads();
  double worst = 0.0;
  const double* H = a.o.feas + b * n * W;
  for (int r = tid; r < rows; r += EP_NT) {
    double s = H[r * W + 2 * n];
    for (int k = 0; k < n; ++k) s += H[r * W + k] * xi[k] + H[r * W + n + k] * xt[k];
    worst = fmax(worst, fabs(s));
  }
  worst = block_max(worst, red);
  if (tid == 0 && a.pt.feas_residual != nullptr) a.pt.feas_residual[b] = worst;
  const double* v0 = a.o.value0 + b * (3 * nn + 2 * n);
  const double* xT = a.pt.x + (b * (T + 1) + T) * n;
  for (int i = tid; i < n; i += EP_NT) {
    double mu = v0[3 * nn + n + i];
    for (int k = 0; k < n; ++k) mu += v0[nn + i * n + k] * xi[k] + v0[2 * nn + i * n + k] * xt[k];
    mu = -mu;
    double g = p.qx1T[b * n + i];
    for (int k = 0; k < n; ++k) g += p.QxxT[b * nn + i * n + k] * xT[k];
    a.pt.mu[b * n + i] = mu;
    const double lt = -g - mu;
    l0[i] = lt;
    a.pt.lam[(b * (T + 1) + T) * n + i] = lt;
  }
  __syncthreads();
  double* cur = l0;
  double* nxt = l1;
  for (int t = T - 1; t >= 0; --t) {
    const int64_t bt = b * T + t;
    const double* x = a.pt.x + (b * (T + 1) + t) * n;
    const double* u = a.pt.u + bt * m;
    const double *Fx = p.Fx + bt * nn, *Qxx = p.Qxx + bt * nn, *Qux = p.Qux + bt * nm;
    for (int i = tid; i < n; i += EP_NT) {
      double s = -p.qx1[bt * n + i];
      for (int k = 0; k < n; ++k) s += Fx[k * n + i] * cur[k] - Qxx[i * n + k] * x[k];
      for (int k = 0; k < m; ++k) s -= Qux[k * n + i] * u[k];
      nxt[i] = s;
      a.pt.lam[(b * (T + 1) + t) * n + i] = s;
    }
    __syncthreads();
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
}

__device__ __forceinline__ double dotv(const double* a, int sa, const double* x, int len) {
  double s0 = 0.0, s1 = 0.0;
  int k = 0;
  for (; k + 1 < len; k += 2) {
    s0 += a[k * sa] * x[k];
    s1 += a[(k + 1) * sa] * x[k + 1];
  }
  if (k < len) s0 += a[k * sa] * x[k];
  return s0 + s1;
}

// objective and the full KKT stack (problem.py:366-420), stage-parallel
__global__ void __launch_bounds__(EP_NT) ep_eval_kernel(EpArgs a) {
  __shared__ double red[32];
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, tid = threadIdx.x;
  const int64_t b = blockIdx.x / a.nch, nn = (int64_t)n * n, nm = (int64_t)n * m;
  const int c = (int)(blockIdx.x % a.nch);
  const int t0 = c * EP_CH, t1 = min(T, t0 + EP_CH);
  double obj = 0.0, kkt = 0.0;
  for (int t = t0; t < t1; ++t) {
    const int64_t bt = b * T + t;
    const double* x = a.pt.x + (b * (T + 1) + t) * n;
    const double* xn = x + n;
    const double* u = a.pt.u + bt * m;
    const double* lam = a.pt.lam + (b * (T + 1) + t) * n;
    const double* lamn = lam + n;
    const double *Fx = p.Fx + bt * nn, *Fu = p.Fu + bt * nm, *Qxx = p.Qxx + bt * nn, *Qux = p.Qux + bt * nm;
    const double* Quu = p.Quu + bt * (int64_t)m * m;
    for (int i = tid; i < n; i += EP_NT) {
      const double g = dotv(Qxx + i * n, 1, x, n);
      const double qx = p.qx1[bt * n + i];
      const double r1 = g + dotv(Qux + i, n, u, m) + qx + lam[i] - dotv(Fx + i, n, lamn, n);
      const double r3 = xn[i] - ((dotv(Fx + i * n, 1, x, n) + dotv(Fu + i * m, 1, u, m)) + p.f1[bt * n + i]);
      kkt = fmax(kkt, fmax(fabs(r1), fabs(r3)));
      obj += x[i] * (0.5 * g + qx);
    }
    for (int i = tid; i < m; i += EP_NT) {
      const double h = dotv(Qux + i * n, 1, x, n);
      const double hu = dotv(Quu + i * m, 1, u, m);
      const double qu = p.qu1[bt * m + i];
      kkt = fmax(kkt, fabs(h + hu + qu - dotv(Fu + i, m, lamn, n)));
      obj += u[i] * (0.5 * hu + h + qu);
    }
  }
  if (t0 == 0)
    for (int i = tid; i < n; i += EP_NT)
      kkt = fmax(kkt, fabs(a.pt.x[b * (T + 1) * n + i] - a.x_init[b * n + i]));
  if (T >= t0 && T < t0 + EP_CH) {   // the chunk holding index T owns the terminal rows
    const double* x = a.pt.x + (b * (T + 1) + T) * n;
    const double* lam = a.pt.lam + (b * (T + 1) + T) * n;
    for (int i = tid; i < n; i += EP_NT) {
      const double g = dotv(p.QxxT + b * nn + i * n, 1, x, n);
      const double qt = p.qx1T[b * n + i];
      obj += x[i] * (0.5 * g + qt);
      kkt = fmax(kkt, fabs(g + qt + lam[i] + a.pt.mu[b * n + i]));
      kkt = fmax(kkt, fabs(x[i] - a.x_term[b * n + i]));
    }
  }
  const double o = block_sum(obj, red);
  const double kv = block_max(kkt, red);
  if (tid == 0) {
    a.part[(b * a.nch + c) * 2] = o;
    a.part[(b * a.nch + c) * 2 + 1] = kv;
  }
}

__global__ void ep_fin_kernel(EpArgs a) {
  __shared__ double red[32];
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, NT = blockDim.x, nch = a.nch;
  const int per = (nch + NT - 1) / NT;
  double obj = 0.0, kkt = 0.0;
  for (int c = tid * per; c < min(nch, (tid + 1) * per); ++c) {
    obj += a.part[(b * nch + c) * 2];
    kkt = fmax(kkt, a.part[(b * nch + c) * 2 + 1]);
  }
  const double o = block_sum(obj, red);
  const double kv = block_max(kkt, red);
  if (tid == 0) {
    a.pt.objective[b] = o;
    a.pt.kkt_inf[b] = kv;
  }
}

}  // namespace

size_t endpoint_scratch_doubles(const plq_problem_t& p) {
  return (size_t)p.B * (p.T + 1) * p.n * p.n + (size_t)p.B * ep_scratch(p.n, p.m);
}

size_t endpoint_eval_doubles(const plq_problem_t& p) {
  const int nch = (p.T + 1 + EP_CH - 1) / EP_CH;
  return (size_t)p.B * nch * 2;
}

int launch_endpoint_maps_mult(const plq_problem_t& p, const plq_endpoint_outputs_t& o, double* ws, cudaStream_t s,
                              int* launches) {
  EpArgs a{};
  a.p = p;
  a.o = o;
  a.Xb = ws;
  a.scratch = ws + (size_t)p.B * (p.T + 1) * p.n * p.n;
  // small states: 4 warps cover every GEMM tile, more CTAs stay resident,
  // and the sequential working sets fit in shared memory
  const int n = p.n, m = p.m, W = 2 * n + 1;
  if (n <= 32) {
    const size_t maps_sm = sizeof(double) * (2 * (size_t)n * W + (size_t)m * W);
    const size_t mult_sm = sizeof(double) * (4 * (size_t)n * W + (size_t)m * W + 4 * (size_t)n * n);
    static unsigned attr = 0;
    if (first_on_device(&attr)) {
      cudaFuncSetAttribute(ep_maps_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(ep_mult_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    ep_maps_kernel<128, true><<<(unsigned)p.B, 128, maps_sm, s>>>(a);
    if (cudaGetLastError() != cudaSuccess) return -1;
    ep_mult_kernel<128, true><<<(unsigned)p.B, 128, mult_sm, s>>>(a);
  } else {
    ep_maps_kernel<EP_NT, false><<<(unsigned)p.B, EP_NT, 0, s>>>(a);
    if (cudaGetLastError() != cudaSuccess) return -1;
    ep_mult_kernel<EP_NT, false><<<(unsigned)p.B, EP_NT, 0, s>>>(a);
  }
  if (cudaGetLastError() != cudaSuccess) return -1;
  *launches += 2;
  return 0;
}

int launch_endpoint_evaluate(const plq_problem_t& p, const plq_endpoint_outputs_t& o, const plq_endpoint_point_t& pt,
                             double* ws, cudaStream_t s, int* launches) {
  EpArgs a{};
  a.p = p;
  a.o = o;
  a.pt = pt;
  a.x_init = pt.x_init ? pt.x_init : p.x_init;
  a.x_term = pt.x_term;
  a.nch = (p.T + 1 + EP_CH - 1) / EP_CH;
  a.part = ws;
  const unsigned grid = (unsigned)(p.B * a.nch);
  ep_point_kernel<<<grid, EP_NT, sizeof(double) * (2 * p.n + 1), s>>>(a);
  if (cudaGetLastError() != cudaSuccess) return -1;
  if (o.feas_rows != nullptr) {
    ep_dual_kernel<<<(unsigned)p.B, EP_NT, sizeof(double) * 4 * p.n, s>>>(a);
    if (cudaGetLastError() != cudaSuccess) return -1;
    ++*launches;
  }
  ep_eval_kernel<<<grid, EP_NT, 0, s>>>(a);
  if (cudaGetLastError() != cudaSuccess) return -1;
  ep_fin_kernel<<<(unsigned)p.B, 256, 0, s>>>(a);
  if (cudaGetLastError() != cudaSuccess) return -1;
  *launches += 3;
  return 0;
}

}  // namespace plq
