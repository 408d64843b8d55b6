// K2/K3 specialized for the small-state configs (compile-time n, m; one warp
// per segment / per problem):
//   * link_seq_kernel: the reference's sequential block Cholesky of the link
//     system (endpoint.solve_block_tridiagonal, endpoint.py:410-438, on
//     (-diag, -sub, rhs) from parallel.py:264-319), one warp per problem --
//     the right shape when J-1 is small (BASELINE configs 0, 1);
//   * recon_small_kernel: the reconstruction loop of parallel.py:485-525 plus
//     the objective / KKT rows of problem.py:366-420, one warp per segment,
//     lane = state row, stage matrices staged in shared memory (odd strides:
//     row-per-lane reads are bank-conflict free) with the next stage
//     prefetched into registers.
#include <stdlib.h>

#include "plq_internal.h"
#include "plq_small.cuh"
#include "plq_tma.cuh"

namespace plq {

namespace {

// ----------------------------------------------------------------------------
// reconstruction

template <int N, int M>
struct RL {
  static constexpr int LN = N + 1, LM = M + 1;   // odd strides (N, M even here)
  static constexpr int FX = 0;                  // N x LN
  static constexpr int FU = FX + N * LN;        // N x LM
  static constexpr int F1 = FU + N * LM;        // N
  static constexpr int QXX = F1 + N;            // N x LN
  static constexpr int QUX = QXX + N * LN;      // M x LN
  static constexpr int QUU = QUX + M * LN;      // M x LM
  static constexpr int QX1 = QUU + M * LM;      // N
  static constexpr int QU1 = QX1 + N;           // M
  static constexpr int KX = QU1 + M;            // M x LN
  static constexpr int KZ = KX + M * LN;        // M x LN
  static constexpr int K1 = KZ + M * LN;        // M
  static constexpr int STAGE = K1 + M;
  // vectors
  static constexpr int X = STAGE, XN = X + N, U = XN + N, KV = U + M, Z = KV + M, A = Z + N, LAM = A + N;
  static constexpr int TOTAL = (LAM + N + 1) & ~1;
  // stage element count (global order Fx|Fu|f1|Qxx|Qux|Quu|qx1|qu1|Kx|Kz|k1)
  static constexpr int SE = 2 * N * N + 2 * N * M + M * M + 2 * N + M + 2 * M * N + M;
};

template <int N, int M>
__device__ __forceinline__ const double* recon_elem(const ReconArgs& A, int64_t st, int e, int& dst, bool last) {
  using S = RL<N, M>;
  constexpr int NN = N * N, NM = N * M;
  const plq_problem_t& p = A.p;
  if (e < NN) { dst = S::FX + (e / N) * S::LN + e % N; return p.Fx + st * NN + e; }
  e -= NN;
  if (e < NM) { dst = S::FU + (e / M) * S::LM + e % M; return p.Fu + st * NM + e; }
  e -= NM;
  if (e < N) { dst = S::F1 + e; return p.f1 + st * N + e; }
  e -= N;
  if (e < NN) { dst = S::QXX + (e / N) * S::LN + e % N; return p.Qxx + st * NN + e; }
  e -= NN;
  if (e < NM) { dst = S::QUX + (e / N) * S::LN + e % N; return p.Qux + st * NM + e; }
  e -= NM;
  if (e < M * M) { dst = S::QUU + (e / M) * S::LM + e % M; return p.Quu + st * M * M + e; }
  e -= M * M;
  if (e < N) { dst = S::QX1 + e; return p.qx1 + st * N + e; }
  e -= N;
  if (e < M) { dst = S::QU1 + e; return p.qu1 + st * M + e; }
  e -= M;
  if (e < NM) { dst = S::KX + (e / N) * S::LN + e % N; return A.Kx + st * NM + e; }
  e -= NM;
  if (e < NM) { dst = S::KZ + (e / N) * S::LN + e % N; return last ? nullptr : A.Kz + st * NM + e; }
  e -= NM;
  dst = S::K1 + e;
  return A.k1 + st * M + e;
}

template <int N, int M>
struct RPrefetch {
  static constexpr int PF = (RL<N, M>::SE + 31) / 32;
  double v[PF];
  __device__ __forceinline__ void load(const ReconArgs& A, int64_t st, int lane, bool last) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int e = lane + 32 * k;
      if (e < RL<N, M>::SE) {
        int d;
        const double* src = recon_elem<N, M>(A, st, e, d, last);
        v[k] = src ? __ldg(src) : 0.0;
      }
    }
  }
  __device__ __forceinline__ void store(const ReconArgs& A, double* sm, int lane) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int e = lane + 32 * k;
      if (e < RL<N, M>::SE) {
        int d;
        recon_elem<N, M>(A, 0, e, d, false);
        sm[d] = v[k];
      }
    }
  }
};

template <int N, int M>
__global__ void __launch_bounds__(32) recon_small_kernel(ReconArgs A) {
  static_assert(N <= 32 && M <= 32, "lane = row");
  using S = RL<N, M>;
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = A.p;
  const int J = p.J, T = p.T, NN = N * N;
  const int lane = threadIdx.x;
  double* x = sm + S::X;
  double* xn = sm + S::XN;
  double* uu = sm + S::U;
  double* kv = sm + S::KV;
  double* z = sm + S::Z;
  double* av = sm + S::A;
  double* lam = sm + S::LAM;
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t total = p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = A.seg_begin + (int)(task % nloc);
    const int lo = p.split_times[j], hi = p.split_times[j + 1], L = hi - lo;
    if (!segment_bounds_ok(p, j)) continue;   // malformed partition (flagged by the sweep)
    const bool last = (j == J - 1);
    if (lane < N) {
      const double a0 = (j == 0) ? p.x_init[b * N + lane] : A.links[(b * (J - 1) + (j - 1)) * N + lane];
      av[lane] = a0;
      x[lane] = a0;
      z[lane] = last ? 0.0 : A.links[(b * (J - 1) + j) * N + lane];
    }
    RPrefetch<N, M> pf;
    pf.load(A, b * T + lo, lane, last);
    pf.store(A, sm, lane);
    __syncwarp();
    double obj = 0.0;      // per-lane partial objective
    double worst = 0.0;    // per-lane KKT partial
    // ---- forward: fold, rollout, stage cost, g/h (parallel.py:495-502)
#pragma unroll 1
    for (int s = 0; s < L; ++s) {
      const int64_t st = b * T + lo + s;
      if (s + 1 < L) pf.load(A, st + 1, lane, last);
      if (lane < M) {
        double kk = sm[S::K1 + lane];
        if (!last) {
          double t = 0.0;
#pragma unroll
          for (int c = 0; c < N; ++c) t += sm[S::KZ + lane * S::LN + c] * z[c];
          kk = t + kk;
        }
        kv[lane] = kk;
        double t = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) t += sm[S::KX + lane * S::LN + c] * x[c];
        uu[lane] = t + kk;
      }
      __syncwarp();
      if (lane < M) {
        A.k[st * M + lane] = kv[lane];
        A.u[st * M + lane] = uu[lane];
      }
      if (lane < N) {
        A.x[(b * (T + 1) + lo + s) * N + lane] = x[lane];
        const double xi = x[lane];
        double t0 = 0.0, t1 = 0.0, fx = 0.0, fu = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) {
          t0 += sm[S::QXX + lane * S::LN + c] * x[c];
          fx += sm[S::FX + lane * S::LN + c] * x[c];
        }
#pragma unroll
        for (int q = 0; q < M; ++q) {
          t1 += sm[S::QUX + q * S::LN + lane] * uu[q];
          fu += sm[S::FU + lane * S::LM + q] * uu[q];
        }
        const double qx = sm[S::QX1 + lane];
        obj += 0.5 * xi * t0 + qx * xi;
        A.gh[st * (N + M) + lane] = (t0 + t1) + qx;
        xn[lane] = (fx + fu) + sm[S::F1 + lane];
      }
      if (lane < M) {
        double t2 = 0.0, t3 = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) t2 += sm[S::QUX + lane * S::LN + c] * x[c];
#pragma unroll
        for (int q = 0; q < M; ++q) t3 += sm[S::QUU + lane * S::LM + q] * uu[q];
        const double ui = uu[lane], qu = sm[S::QU1 + lane];
        obj += 0.5 * ui * t3 + ui * t2 + qu * ui;
        A.gh[st * (N + M) + N + lane] = (t2 + t3) + qu;
      }
      __syncwarp();
      if (lane < N) x[lane] = xn[lane];
      if (s + 1 < L) pf.store(A, sm, lane);
      __syncwarp();
    }
    // ---- multiplier seed (parallel.py:505-515)
    if (last) {
      if (lane < N) {
        A.x[(b * (T + 1) + T) * N + lane] = x[lane];
        double t = 0.0;
        const double* QT = p.QxxT + b * NN + lane * N;
#pragma unroll
        for (int c = 0; c < N; ++c) t += QT[c] * x[c];
        const double q1 = p.qx1T[b * N + lane];
        obj += 0.5 * x[lane] * t + q1 * x[lane];
        const double g = t + q1;
        lam[lane] = -g;
        A.lam[(b * (T + 1) + T) * N + lane] = -g;
        worst = fmax(worst, fabs(g + -g));
      }
    } else {
      if (lane < N) {
        A.xend[(b * J + j) * N + lane] = x[lane];
        const double* vf = A.vf0 + (b * J + j) * (int64_t)(3 * NN + 2 * N);
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) {
          t0 += vf[NN + lane * N + c] * av[c];
          t1 += vf[2 * NN + lane * N + c] * z[c];
        }
        const double mu = -((t0 + t1) + vf[3 * NN + N + lane]) - (A.mu_corr && A.feas_rows[b * J + j] > 0 ? A.mu_corr[(b * J + j) * N + lane] : 0.0);
        A.mu_left[(b * (J - 1) + j) * N + lane] = mu;
        lam[lane] = -mu;
      }
    }
    __syncwarp();
    // ---- backward multiplier recursion (parallel.py:518-523) + interior KKT rows
#pragma unroll 1
    for (int s = L - 1; s >= 0; --s) {
      const int64_t st = b * T + lo + s;
      const bool interior = last || (s < L - 1);
      double ln = 0.0;
      if (lane < N) {
        const double* Fx = p.Fx + st * NN;
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) t += __ldg(Fx + k * N + lane) * lam[k];
        const double g = A.gh[st * (N + M) + lane];
        ln = t - g;
        A.lam[(b * (T + 1) + lo + s) * N + lane] = ln;
        if (interior) worst = fmax(worst, fabs((g + ln) - t));
      }
      if (lane < M && interior) {
        const double* Fu = p.Fu + st * N * M;
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) t += __ldg(Fu + k * M + lane) * lam[k];
        worst = fmax(worst, fabs(A.gh[st * (N + M) + N + lane] - t));
      }
      __syncwarp();
      if (lane < N) lam[lane] = ln;
      __syncwarp();
    }
    if (j > 0 && lane < N) A.lambda_right[(b * (J - 1) + (j - 1)) * N + lane] = lam[lane];
    obj = warp_sum(obj);
    worst = warp_max(worst);
    if (lane == 0) {
      A.part[(b * J + j) * 3 + 0] = obj;
      A.part[(b * J + j) * 3 + 1] = worst;
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// whole-segment variant: the segment's 11 per-stage fields are contiguous
// L-stage blocks in global memory, so one bulk copy per field (TMA 1-D,
// cp.async.bulk) stages the entire segment in shared memory; the forward
// rollout and the backward multiplier recursion then run from smem, and g/h
// stay on chip.

template <int N, int M>
__device__ __forceinline__ void seg_issue(const ReconArgs& A, double* buf, uint64_t* bar, int64_t s0, int L,
                                          const double* vf, bool endpoint) {
  constexpr int NN = N * N, NM = N * M, MM = M * M;
  const plq_problem_t& p = A.p;
  fence_proxy_async();
  const uint32_t l8 = (uint32_t)L * 8u;
  const uint32_t vbytes = endpoint ? 8u * (2 * NN + 2 * N) : 0u;
  (void)MM;
  mbar_arrive_tx(bar, l8 * (NN + NM + N) + vbytes);   // the fields below
  double* d = buf;
  bulk_g2s(d, p.Fx + s0 * NN, l8 * NN, bar);
  d += L * NN;
  bulk_g2s(d, p.Fu + s0 * NM, l8 * NM, bar);
  d += L * NM;
  bulk_g2s(d, p.f1 + s0 * N, l8 * N, bar);
  d += L * N;
  if (endpoint) bulk_g2s(d, vf + NN, vbytes, bar);   // Vzx0, Vzz0, vx10, vz10
}

// Row-fused reconstruction for 2n + 2m = 32 (n = 12, m = 4): in each
// dot-product pass every lane owns one row of a different matrix, e.g. pass 1
// computes Fx x | Kx x | Qxx x | Qux x on lanes 0-11 | 12-15 | 16-27 | 28-31.
// Only Fx, Fu, f1 (reused by the backward pass) are bulk-staged for the whole
// segment; the policy / cost rows a lane owns are register-prefetched one
// stage ahead from global, which keeps ~17 KB of smem per warp (occupancy).
template <int N, int M, int LMAX>
__global__ void __launch_bounds__(32) recon_seg_kernel(ReconArgs A) {
  static_assert(2 * N + 2 * M == 32, "row-fused lane map");
  constexpr int NN = N * N, NM = N * M, MM = M * M;
  constexpr int BUF = LMAX * (NN + NM + N) + 2 * NN + 2 * N;
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = A.p;
  const int J = p.J, T = p.T;
  const int lane = threadIdx.x;
  double* buf = sm;
  double* gh = sm + BUF;                 // LMAX x (N+M)
  double* kv = gh + LMAX * (N + M);      // LMAX x M folded offsets
  double* x = kv + LMAX * M;             // N
  double* xn = x + N;                    // N
  double* uu = xn + N;                   // M
  double* z = uu + M;                    // N
  double* av = z + N;                    // N
  double* lam = av + N;                  // N
  uint64_t* bar = reinterpret_cast<uint64_t*>(lam + N);
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  uint32_t phase = 0;
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t total = p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = A.seg_begin + (int)(task % nloc);
    const int lo = p.split_times[j], L = p.split_times[j + 1] - lo;
    if (L < 1 || L > LMAX) continue;     // malformed partition: flagged by the sweep, buffers sized for LMAX
    const bool last = (j == J - 1);
    const int64_t s0 = b * T + lo;
    const double* vfg = A.vf0 + (b * J + j) * (int64_t)(3 * NN + 2 * N);
    if (lane == 0) seg_issue<N, M>(A, buf, bar, s0, L, vfg, !last);
    const double* FX = buf;
    const double* FU = FX + L * NN;
    const double* F1 = FU + L * NM;
    const double* KZ = A.Kz + s0 * NM;   // global (fold)
    const double* K1 = A.k1 + s0 * M;
    const double* VZX = F1 + L * N;      // endpoint segments only
    const double* VZZ = VZX + NN;
    const double* VZ1 = VZZ + NN + N;
    if (lane < N) {
      const double a0 = (j == 0) ? p.x_init[b * N + lane] : A.links[(b * (J - 1) + (j - 1)) * N + lane];
      av[lane] = a0;
      x[lane] = a0;
      z[lane] = last ? 0.0 : A.links[(b * (J - 1) + j) * N + lane];
    }
    __syncwarp();
    // fold k = Kz z + k1 for every stage at once (parallel.py:495), from
    // global while the bulk copies land
    for (int r = lane; r < L * M; r += 32) {
      const double* kz = KZ + r * N;
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) t += kz[c] * z[c];
      kv[r] = t + K1[r];
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    __syncwarp();
    double obj = 0.0, worst = 0.0;
    // lane roles of the two forward passes
    const int grp = lane < N ? 0 : (lane < N + M ? 1 : (lane < 2 * N + M ? 2 : 3));
    const int row = grp == 0 ? lane : (grp == 1 ? lane - N : (grp == 2 ? lane - N - M : lane - 2 * N - M));
    // this lane's pass-1 row (Kx | Qxx | Qux), pass-2 vector (Qux col | Quu
    // row) and scalar (qx1 | qu1) of a stage, straight from global
    double pr[N], pq[M], ps = 0.0;
    auto fetch = [&](int s, double* r, double* v, double& sc) {
      const int64_t st = s0 + s;
      if (grp == 1) {
#pragma unroll
        for (int c = 0; c < N; ++c) r[c] = A.Kx[st * NM + row * N + c];
      } else if (grp == 2) {
#pragma unroll
        for (int c = 0; c < N; ++c) r[c] = p.Qxx[st * NN + row * N + c];
#pragma unroll
        for (int q = 0; q < M; ++q) v[q] = p.Qux[st * NM + q * N + row];
        sc = p.qx1[st * N + row];
      } else if (grp == 3) {
#pragma unroll
        for (int c = 0; c < N; ++c) r[c] = p.Qux[st * NM + row * N + c];
#pragma unroll
        for (int q = 0; q < M; ++q) v[q] = p.Quu[st * MM + row * M + q];
        sc = p.qu1[st * M + row];
      }
    };
    fetch(0, pr, pq, ps);
#pragma unroll 1
    for (int s = 0; s < L; ++s) {
      const int64_t st = s0 + s;
      double nr[N], nq[M], ns = 0.0;
      if (s + 1 < L) fetch(s + 1, nr, nq, ns);
      if (grp == 0) {
#pragma unroll
        for (int c = 0; c < N; ++c) pr[c] = FX[s * NN + row * N + c];
      }
      // pass 1: Fx x | Kx x | Qxx x | Qux x
      double t = 0.0, t_ = 0.0;
#pragma unroll
      for (int c = 0; c < N; c += 2) {
        t += pr[c] * x[c];
        t_ += pr[c + 1] * x[c + 1];
      }
      t += t_;
      if (grp == 1) {
        const double kk = kv[s * M + row];
        const double uv = t + kk;
        uu[row] = uv;
        A.k[st * M + row] = kk;
        A.u[st * M + row] = uv;
      }
      __syncwarp();
      // pass 2: Fu u | - | Qux' u | Quu u
      double t2 = 0.0;
      if (grp == 0) {
#pragma unroll
        for (int q = 0; q < M; ++q) t2 += FU[s * NM + row * M + q] * uu[q];
        xn[row] = (t + t2) + F1[s * N + row];
      } else if (grp == 2) {
#pragma unroll
        for (int q = 0; q < M; ++q) t2 += pq[q] * uu[q];
        const double xi = x[row], qx = ps;
        gh[s * (N + M) + row] = (t + t2) + qx;
        obj += 0.5 * xi * t + qx * xi;
        A.x[(b * (T + 1) + lo + s) * N + row] = xi;
      } else if (grp == 3) {
#pragma unroll
        for (int q = 0; q < M; ++q) t2 += pq[q] * uu[q];
        const double ui = uu[row], qu = ps;
        gh[s * (N + M) + N + row] = (t + t2) + qu;
        obj += 0.5 * ui * t2 + ui * t + qu * ui;
      }
      __syncwarp();
      if (lane < N) x[lane] = xn[lane];
      __syncwarp();
#pragma unroll
      for (int c = 0; c < N; ++c) pr[c] = nr[c];
#pragma unroll
      for (int q = 0; q < M; ++q) pq[q] = nq[q];
      ps = ns;
    }
    // g/h of the link stage feed the boundary kernel
    if (lane < N + M) A.gh[(s0 + L - 1) * (N + M) + lane] = gh[(L - 1) * (N + M) + lane];
    // ---- multiplier seed (parallel.py:505-515)
    if (last) {
      if (lane < N) {
        A.x[(b * (T + 1) + T) * N + lane] = x[lane];
        double tt = 0.0;
        const double* QT = p.QxxT + b * NN + lane * N;
#pragma unroll
        for (int c = 0; c < N; ++c) tt += QT[c] * x[c];
        const double q1 = p.qx1T[b * N + lane];
        obj += 0.5 * x[lane] * tt + q1 * x[lane];
        const double g = tt + q1;
        lam[lane] = -g;
        A.lam[(b * (T + 1) + T) * N + lane] = -g;
        worst = fmax(worst, fabs(g + -g));
      }
    } else {
      // mu = -(Vzx0 a + Vzz0 z + vz10): lanes 0-11 Vzx0 a, lanes 16-27 Vzz0 z
      double tv = 0.0;
      const bool hi = lane >= 16 && lane < 16 + N;
      const int rr = hi ? lane - 16 : lane;
      if (lane < N || hi) {
        const double* mrow = hi ? VZZ + rr * N : VZX + rr * N;
        const double* vec = hi ? z : av;
#pragma unroll
        for (int c = 0; c < N; ++c) tv += mrow[c] * vec[c];
      }
      const double tz = __shfl_down_sync(0xffffffffu, tv, 16);
      if (lane < N) {
        A.xend[(b * J + j) * N + lane] = x[lane];
        const double mu = -((tv + tz) + VZ1[lane]) - (A.mu_corr && A.feas_rows[b * J + j] > 0 ? A.mu_corr[(b * J + j) * N + lane] : 0.0);
        A.mu_left[(b * (J - 1) + j) * N + lane] = mu;
        lam[lane] = -mu;
      }
    }
    __syncwarp();
    // ---- backward multipliers (parallel.py:518-523) + interior KKT rows:
    // lanes 0-11 Fx' lam, lanes 12-15 Fu' lam
#pragma unroll 1
    for (int s = L - 1; s >= 0; --s) {
      const bool interior = last || (s < L - 1);
      double tb = 0.0, tb_ = 0.0;
      if (lane < N + M) {
        const double* col = lane < N ? FX + s * NN + lane : FU + s * NM + (lane - N);
        const int stride = lane < N ? N : M;
#pragma unroll
        for (int k = 0; k < N; k += 2) {
          tb += col[k * stride] * lam[k];
          tb_ += col[(k + 1) * stride] * lam[k + 1];
        }
        tb += tb_;
      }
      double ln = 0.0;
      if (lane < N) {
        const double g = gh[s * (N + M) + lane];
        ln = tb - g;
        A.lam[(b * (T + 1) + lo + s) * N + lane] = ln;
        if (interior) worst = fmax(worst, fabs((g + ln) - tb));
      } else if (lane < N + M && interior) {
        worst = fmax(worst, fabs(gh[s * (N + M) + lane] - tb));
      }
      __syncwarp();
      if (lane < N) lam[lane] = ln;
      __syncwarp();
    }
    if (j > 0 && lane < N) A.lambda_right[(b * (J - 1) + (j - 1)) * N + lane] = lam[lane];
    obj = warp_sum(obj);
    worst = warp_max(worst);
    if (lane == 0) {
      A.part[(b * J + j) * 3 + 0] = obj;
      A.part[(b * J + j) * 3 + 1] = worst;
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// ring variant for longer segments / larger n (BASELINE config 2: n = 32,
// m = 8, L = 64): a CTA per segment, stages streamed through an RS-slot ring
// of bulk copies (forward: all 11 fields; backward: Fx, Fu only), g/h kept on
// chip for the whole segment, row-fused passes over the CTA's threads.

template <int N, int M>
struct RingL {
  static constexpr int NN = N * N, NM = N * M, MM = M * M;
  static constexpr int SLOT = 2 * NN + 4 * NM + MM + 2 * N + 2 * M;   // one stage, forward fields
  static constexpr int FX = 0, FU = NN, F1 = FU + NM, QXX = F1 + N, QUX = QXX + NN, QUU = QUX + NM,
                       QX1 = QUU + MM, QU1 = QX1 + N, KX = QU1 + M, KZ = KX + NM, K1 = KZ + NM;
  static constexpr uint32_t FWD_BYTES = 8u * SLOT, BWD_BYTES = 8u * (NN + NM);
};

template <int N, int M>
__device__ __forceinline__ void ring_issue_fwd(const ReconArgs& A, double* slot, uint64_t* bar, int64_t st) {
  using R = RingL<N, M>;
  constexpr int NN = N * N, NM = N * M, MM = M * M;
  const plq_problem_t& p = A.p;
  fence_proxy_async();
  mbar_arrive_tx(bar, R::FWD_BYTES);
  bulk_g2s(slot + R::FX, p.Fx + st * NN, 8u * NN, bar);
  bulk_g2s(slot + R::FU, p.Fu + st * NM, 8u * NM, bar);
  bulk_g2s(slot + R::F1, p.f1 + st * N, 8u * N, bar);
  bulk_g2s(slot + R::QXX, p.Qxx + st * NN, 8u * NN, bar);
  bulk_g2s(slot + R::QUX, p.Qux + st * NM, 8u * NM, bar);
  bulk_g2s(slot + R::QUU, p.Quu + st * MM, 8u * MM, bar);
  bulk_g2s(slot + R::QX1, p.qx1 + st * N, 8u * N, bar);
  bulk_g2s(slot + R::QU1, p.qu1 + st * M, 8u * M, bar);
  bulk_g2s(slot + R::KX, A.Kx + st * NM, 8u * NM, bar);
  bulk_g2s(slot + R::KZ, A.Kz + st * NM, 8u * NM, bar);
  bulk_g2s(slot + R::K1, A.k1 + st * M, 8u * M, bar);
}

template <int N, int M>
__device__ __forceinline__ void ring_issue_bwd(const ReconArgs& A, double* slot, uint64_t* bar, int64_t st) {
  using R = RingL<N, M>;
  constexpr int NN = N * N, NM = N * M;
  fence_proxy_async();
  mbar_arrive_tx(bar, R::BWD_BYTES);
  bulk_g2s(slot + R::FX, A.p.Fx + st * NN, 8u * NN, bar);
  bulk_g2s(slot + R::FU, A.p.Fu + st * NM, 8u * NM, bar);
}

template <int N, int M, int NT, int RS>
__global__ void __launch_bounds__(NT) recon_ring_kernel(ReconArgs A) {
  // large n: the segment-start blocks (Vzx0, Vzz0, vz10) are read from global
  // memory once per segment instead of being staged
  constexpr bool VFG = N >= 64;
  using R = RingL<N, M>;
  constexpr int NN = N * N, NM = N * M, MM = M * M;
  static_assert(2 * N + 3 * M <= NT, "row-fused passes need one thread per row");
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = A.p;
  const int J = p.J, T = p.T, tid = threadIdx.x;
  const int LMAX = p.max_seg_len;
  double* ring = sm;                                  // RS x SLOT
  double* vfb = ring + RS * R::SLOT;                  // Vzx0, Vzz0, vx10, vz10 (2NN + 2N) unless VFG
  double* gh = vfb + (VFG ? 0 : 2 * NN + 2 * N);      // LMAX x (N+M)
  double* x = gh + (size_t)LMAX * (N + M);
  double* xn = x + N;
  double* uu = xn + N;
  double* z = uu + M;
  double* av = z + N;
  double* lam = av + N;
  double* tf = lam + N;    // pass-1 results
  double* tu = tf + N;
  double* t0 = tu + M;
  double* t2 = t0 + N;
  double* tk = t2 + M;
  double* red = tk + M;    // NT / 32 doubles
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + NT / 32 + ((N + M) & 1));
  uint64_t* vbar = bars + RS;
  if (tid == 0) {
    for (int k = 0; k <= RS; ++k) mbar_init(bars + k, 1);
  }
  __syncthreads();
  uint32_t ph[RS + 1];
#pragma unroll
  for (int k = 0; k <= RS; ++k) ph[k] = 0u;
  // thread roles of pass 1: Fx x | Kx x | Qxx x | Qux x | Kz z
  const int role = tid < N ? 0 : (tid < N + M ? 1 : (tid < 2 * N + M ? 2 : (tid < 2 * N + 2 * M ? 3 : (tid < 2 * N + 3 * M ? 4 : 5))));
  const int row = role == 0 ? tid : (role == 1 ? tid - N : (role == 2 ? tid - N - M : (role == 3 ? tid - 2 * N - M : tid - 2 * N - 2 * M)));
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t total = p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = A.seg_begin + (int)(task % nloc);
    const int lo = p.split_times[j], L = p.split_times[j + 1] - lo;
    if (L < 1 || L > LMAX) continue;     // malformed partition: flagged by the sweep; gh holds LMAX stages
    const bool last = (j == J - 1);
    const int64_t s0 = b * T + lo;
    const double* vfg = A.vf0 + (b * J + j) * (int64_t)(3 * NN + 2 * N);
    if (tid == 0) {
      for (int k = 0; k < RS && k < L; ++k) ring_issue_fwd<N, M>(A, ring + k * R::SLOT, bars + k, s0 + k);
      if (!last && !VFG) {
        fence_proxy_async();
        mbar_arrive_tx(vbar, 8u * (2 * NN + 2 * N));
        bulk_g2s(vfb, vfg + NN, 8u * (2 * NN + 2 * N), vbar);
      }
    }
    if (tid < N) {
      const double a0 = (j == 0) ? p.x_init[b * N + tid] : A.links[(b * (J - 1) + (j - 1)) * N + tid];
      av[tid] = a0;
      x[tid] = a0;
      z[tid] = last ? 0.0 : A.links[(b * (J - 1) + j) * N + tid];
    }
    __syncthreads();
    double obj = 0.0, worst = 0.0;
    // ---- forward
#pragma unroll 1
    for (int s = 0; s < L; ++s) {
      const int slot = s % RS;
      const double* sl = ring + slot * R::SLOT;
      mbar_wait(bars + slot, ph[slot]);
      ph[slot] ^= 1u;
      const int64_t st = s0 + s;
      if (role < 5) {
        const double* rp = role == 0 ? sl + R::FX + row * N
                                     : (role == 1 ? sl + R::KX + row * N
                                                  : (role == 2 ? sl + R::QXX + row * N
                                                               : (role == 3 ? sl + R::QUX + row * N : sl + R::KZ + row * N)));
        const double* vec = role == 4 ? z : x;
        double t = 0.0, t_ = 0.0;
#pragma unroll 8
        for (int c = 0; c < N; c += 2) {
          t += rp[c] * vec[c];
          t_ += rp[c + 1] * vec[c + 1];
        }
        t += t_;
        double* dst = role == 0 ? tf : (role == 1 ? tu : (role == 2 ? t0 : (role == 3 ? t2 : tk)));
        dst[row] = t;
      }
      __syncthreads();
      if (tid < M) {
        const double kk = tk[tid] + sl[R::K1 + tid];
        const double uv = tu[tid] + kk;
        uu[tid] = uv;
        A.k[st * M + tid] = kk;
        A.u[st * M + tid] = uv;
      }
      __syncthreads();
      if (tid < N) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) t += sl[R::FU + tid * M + q] * uu[q];
        xn[tid] = (tf[tid] + t) + sl[R::F1 + tid];
      } else if (tid < 2 * N) {
        const int i = tid - N;
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) t += sl[R::QUX + q * N + i] * uu[q];
        const double xi = x[i], qx = sl[R::QX1 + i];
        gh[s * (N + M) + i] = (t0[i] + t) + qx;
        obj += 0.5 * xi * t0[i] + qx * xi;
        A.x[(b * (T + 1) + lo + s) * N + i] = xi;
      } else if (tid < 2 * N + M) {
        const int u = tid - 2 * N;
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) t += sl[R::QUU + u * M + q] * uu[q];
        const double ui = uu[u], qu = sl[R::QU1 + u];
        gh[s * (N + M) + N + u] = (t2[u] + t) + qu;
        obj += 0.5 * ui * t + ui * t2[u] + qu * ui;
      }
      __syncthreads();
      if (tid == 0 && s + RS < L) ring_issue_fwd<N, M>(A, ring + slot * R::SLOT, bars + slot, st + RS);
      if (tid < N) x[tid] = xn[tid];
      __syncthreads();
    }
    if (tid < N + M) A.gh[(s0 + L - 1) * (N + M) + tid] = gh[(L - 1) * (N + M) + tid];
    // backward prologue: Fx, Fu of the last RS stages
    if (tid == 0)
      for (int k = 0; k < RS && k < L; ++k) ring_issue_bwd<N, M>(A, ring + k * R::SLOT, bars + k, s0 + L - 1 - k);
    // ---- multiplier seed
    if (last) {
      if (tid < N) {
        A.x[(b * (T + 1) + T) * N + tid] = x[tid];
        double t = 0.0;
        const double* QT = p.QxxT + b * NN + tid * N;
        for (int c = 0; c < N; ++c) t += QT[c] * x[c];
        const double q1 = p.qx1T[b * N + tid];
        obj += 0.5 * x[tid] * t + q1 * x[tid];
        const double g = t + q1;
        lam[tid] = -g;
        A.lam[(b * (T + 1) + T) * N + tid] = -g;
        worst = fmax(worst, fabs(g + -g));
      }
    } else {
      const double* vsrc = VFG ? vfg + NN : vfb;
      if (!VFG) {
        mbar_wait(vbar, ph[RS]);
        ph[RS] ^= 1u;
      }
      if (tid < N) {
        A.xend[(b * J + j) * N + tid] = x[tid];
        double t0v = 0.0, t1v = 0.0;
        for (int c = 0; c < N; ++c) {
          t0v += vsrc[tid * N + c] * av[c];
          t1v += vsrc[NN + tid * N + c] * z[c];
        }
        const double mu = -((t0v + t1v) + vsrc[2 * NN + N + tid]) - (A.mu_corr && A.feas_rows[b * J + j] > 0 ? A.mu_corr[(b * J + j) * N + tid] : 0.0);
        A.mu_left[(b * (J - 1) + j) * N + tid] = mu;
        lam[tid] = -mu;
      }
    }
    __syncthreads();
    // ---- backward multipliers + interior KKT rows: threads < N Fx' lam, N..N+M-1 Fu' lam
#pragma unroll 1
    for (int k = 0; k < L; ++k) {
      const int s = L - 1 - k;
      const int slot = k % RS;
      const double* sl = ring + slot * R::SLOT;
      mbar_wait(bars + slot, ph[slot]);
      ph[slot] ^= 1u;
      const bool interior = last || (s < L - 1);
      double tb = 0.0, ln = 0.0;
      if (tid < N + M) {
        const double* col = tid < N ? sl + R::FX + tid : sl + R::FU + (tid - N);
        const int stride = tid < N ? N : M;
        double t_ = 0.0;
#pragma unroll 8
        for (int q = 0; q < N; q += 2) {
          tb += col[q * stride] * lam[q];
          t_ += col[(q + 1) * stride] * lam[q + 1];
        }
        tb += t_;
      }
      if (tid < N) {
        const double g = gh[s * (N + M) + tid];
        ln = tb - g;
        A.lam[(b * (T + 1) + lo + s) * N + tid] = ln;
        if (interior) worst = fmax(worst, fabs((g + ln) - tb));
      } else if (tid < N + M && interior) {
        worst = fmax(worst, fabs(gh[s * (N + M) + tid] - tb));
      }
      __syncthreads();
      if (tid == 0 && k + RS < L) ring_issue_bwd<N, M>(A, ring + slot * R::SLOT, bars + slot, s0 + s - RS);
      if (tid < N) lam[tid] = ln;
      __syncthreads();
    }
    if (j > 0 && tid < N) A.lambda_right[(b * (J - 1) + (j - 1)) * N + tid] = lam[tid];
    obj = block_sum(obj, red);
    worst = block_max(worst, red);
    if (tid == 0) {
      A.part[(b * J + j) * 3 + 0] = obj;
      A.part[(b * J + j) * 3 + 1] = worst;
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------
// sequential link solve, one warp per problem

// One warp per problem: the reference's block Cholesky (endpoint.py:410-438).
// The segment-start value blocks stream through a 3-slot ring of bulk copies
// (block i+2 in flight while step i computes on blocks i, i+1), pivot /
// right-hand-side blocks ping-pong in smem, the pivot block is factored
// element-parallel across the warp (reciprocal pivots kept), only X_i goes to
// global.  The residual pass streams the blocks again (L2-resident).
template <int N>
__global__ void __launch_bounds__(32, 12) link_seq_kernel(plq_problem_t p, const double* vf0, double* links,
                                                     double* link_residual, int32_t* status, double* Xs) {
  constexpr int LD = N + 1, NN = N * N, VS = 3 * NN + 2 * N, NS = 3;
  constexpr int NTRI = N * (N + 1) / 2;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x;
  const int J = p.J, K = J - 1;
  double* RING = sm;                     // NS x VS
  double* Pm = RING + NS * VS;           // N x LD
  double* R0 = Pm + N * LD;              // N x LD  ping
  double* R1 = R0 + N * LD;              // N x LD  pong
  double* dv = R1 + N * LD;              // K x N
  double* idg = dv + K * N;              // N
  unsigned char* tri = reinterpret_cast<unsigned char*>(idg + N);   // NTRI (ri, ci) pairs
  uint64_t* bar = reinterpret_cast<uint64_t*>(idg + N + (2 * NTRI + 7) / 8 + 1);
  for (int e = lane; e < NTRI; e += 32) {
    int ri = 0;
    while ((ri + 1) * (ri + 2) / 2 <= e) ++ri;
    tri[2 * e] = (unsigned char)ri;
    tri[2 * e + 1] = (unsigned char)(e - ri * (ri + 1) / 2);
  }
  if (lane < NS) mbar_init(bar + lane, 1);
  __syncwarp();
  uint32_t phases = 0;   // bit s: parity of slot s's next completion
  auto issue = [&](const double* src, int blk) {
    if (lane == 0) {
      const int s = blk % NS;
      fence_proxy_async();
      mbar_arrive_tx(bar + s, (uint32_t)(VS * 8));
      bulk_g2s(RING + s * VS, src + (int64_t)blk * VS, (uint32_t)(VS * 8), bar + s);
    }
  };
  auto wait = [&](int blk) {
    const int s = blk % NS;
    mbar_wait(bar + s, (phases >> s) & 1u);
    phases ^= 1u << s;
  };
  for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
    const double* src = vf0 + b * (int64_t)J * VS;
    issue(src, 0);
    issue(src, 1);
    double* X = Xs + b * (int64_t)K * NN;
    const double* xi = p.x_init + b * N;
    int bad = 0;
    double* R = R0;
    double* RP = R1;
    wait(0);
    for (int i = 0; i < K; ++i) {
      if (i + 2 < J) issue(src, i + 2);
      wait(i + 1);
      const double* left = RING + (i % NS) * VS;
      const double* right = RING + ((i + 1) % NS) * VS;
      // P = Vzz0_i + Vxx0_{i+1};  R = [S_i' | b_i],  S_i = Vzx0_{i+1}
      for (int idx = lane; idx < NN; idx += 32) {
        const int r = idx / N, c = idx % N;
        Pm[r * LD + c] = left[2 * NN + idx] + right[idx];
        R[r * LD + c] = (i + 1 < K) ? right[NN + c * N + r] : 0.0;
      }
      if (lane < N) {
        double v = -left[3 * NN + N + lane] + -right[3 * NN + lane];
        if (i == 0) {
          double t = 0.0;
#pragma unroll
          for (int c = 0; c < N; ++c) t += left[NN + lane * N + c] * xi[c];
          v += -t;
        }
        R[lane * LD + N] = v;
      }
      __syncwarp();
      if (i > 0) {
        // P -= S_{i-1} X_{i-1};  g -= S_{i-1} d_{i-1}   (S_{i-1} = Vzx0_i, left block)
        for (int idx = lane; idx < NN; idx += 32) {
          const int r = idx / N, c = idx % N;
          double t = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) t += left[NN + r * N + k] * RP[k * LD + c];
          Pm[r * LD + c] -= t;
        }
        if (lane < N) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) t += left[NN + lane * N + k] * RP[k * LD + N];
          R[lane * LD + N] -= t;
        }
        __syncwarp();
      }
      // Cholesky of P with unscaled pivot columns (one reciprocal and one
      // barrier per column, P_rc -= P_rk P_ck / P_kk), element-parallel
      // trailing updates; the columns are scaled by 1/sqrt(pivot) in one
      // pass at the end.  Reciprocal pivots in idg.
      for (int k = 0; k < N; ++k) {
        const double dkk = Pm[k * LD + k];
        bad |= !(dkk > 0.0);
        const double rk = 1.0 / (dkk > 0.0 ? dkk : 1.0);
        const int s = N - 1 - k;   // trailing triangle (rows/cols k+1..N-1)
        for (int e = lane; e < s * (s + 1) / 2; e += 32) {
          const int r = k + 1 + tri[2 * e], c = k + 1 + tri[2 * e + 1];
          Pm[r * LD + c] -= (Pm[r * LD + k] * rk) * Pm[c * LD + k];
        }
        __syncwarp();
      }
      {
        // off-diagonal entries first (they read the unscaled pivots), then the diagonal
        for (int e = lane; e < N * (N - 1) / 2; e += 32) {
          const int r = 1 + tri[2 * e], c = tri[2 * e + 1];   // strict lower triangle
          const double pk = Pm[c * LD + c];
          Pm[r * LD + c] *= rsqrt(pk > 0.0 ? pk : 1.0);
        }
        __syncwarp();
        if (lane < N) {
          const double pk = Pm[lane * LD + lane];
          const double ir = rsqrt(pk > 0.0 ? pk : 1.0);
          Pm[lane * LD + lane] = pk * ir;
          idg[lane] = ir;
        }
        __syncwarp();
      }
      // R <- P^{-1} R (lane per column; N+1 columns)
      for (int col = lane; col < N + 1; col += 32) {
        double xv[N];
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double v = R[r * LD + col];
#pragma unroll
          for (int k = 0; k < r; ++k) v -= Pm[r * LD + k] * xv[k];
          xv[r] = v * idg[r];
        }
#pragma unroll
        for (int r = N - 1; r >= 0; --r) {
          double v = xv[r];
#pragma unroll
          for (int k = r + 1; k < N; ++k) v -= Pm[k * LD + r] * xv[k];
          xv[r] = v * idg[r];
        }
#pragma unroll
        for (int r = 0; r < N; ++r) R[r * LD + col] = xv[r];
      }
      __syncwarp();
      for (int idx = lane; idx < NN; idx += 32) X[i * NN + idx] = R[(idx / N) * LD + idx % N];
      if (lane < N) dv[i * N + lane] = R[lane * LD + N];
      double* t = R;
      R = RP;
      RP = t;
      __syncwarp();
    }
    // back substitution: out_{K-1} = d_{K-1}; out_i = d_i - X_i out_{i+1}  (in place in dv)
    for (int i = K - 2; i >= 0; --i) {
      if (lane < N) {
        double t = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) t += X[i * NN + lane * N + c] * dv[(i + 1) * N + c];
        dv[i * N + lane] -= t;
      }
      __syncwarp();
    }
    double* out = links + b * (int64_t)K * N;
    for (int idx = lane; idx < K * N; idx += 32) out[idx] = dv[idx];
    // residual of the link equations at the solution (parallel.py:273-282),
    // blocks streamed again through the ring
    __syncwarp();
    issue(src, 0);
    issue(src, 1);
    wait(0);
    double worst = 0.0;
    for (int i = 0; i < K; ++i) {
      if (i + 2 < J) issue(src, i + 2);
      wait(i + 1);
      const double* left = RING + (i % NS) * VS;
      const double* right = RING + ((i + 1) % NS) * VS;
      if (lane < N) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) s += (left[2 * NN + lane * N + c] + right[lane * N + c]) * dv[i * N + c];
        if (i >= 1) {
#pragma unroll
          for (int c = 0; c < N; ++c) s += left[NN + lane * N + c] * dv[(i - 1) * N + c];
        }
        if (i + 1 < K) {
#pragma unroll
          for (int c = 0; c < N; ++c) s += right[NN + c * N + lane] * dv[(i + 1) * N + c];
        }
        double rhs = -left[3 * NN + N + lane] + -right[3 * NN + lane];
        if (i == 0) {
          double t = 0.0;
#pragma unroll
          for (int c = 0; c < N; ++c) t += left[NN + lane * N + c] * xi[c];
          rhs += -t;
        }
        worst = fmax(worst, fabs(s - rhs));
      }
      __syncwarp();
    }
    worst = warp_max(worst);
    if (lane == 0) {
      link_residual[b] = worst;
      if (bad && status[b * J] == 0) status[b * J] = PLQ_STATUS_LINK_SINGULAR;
    }
    __syncwarp();
  }
}

int sms_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <int N, int M, int LMAX>
int launch_recon_seg(const ReconArgs& a, cudaStream_t s) {
  constexpr int BUF = LMAX * (N * N + N * M + N) + 2 * N * N + 2 * N;
  const size_t smem = sizeof(double) * (BUF + LMAX * (N + M) + LMAX * M + 5 * N + M + 4);
  auto kern = recon_seg_kernel<N, M, LMAX>;
  static unsigned attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  const int64_t tasks = a.p.B * (int64_t)(a.seg_end - a.seg_begin);
  // persistent grid: exactly the resident CTAs (registers and shared memory
  // both counted), so no CTA's task stride starts after the others finish
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, smem);
  const int64_t cap = (int64_t)sms_count() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(tasks < cap ? tasks : cap);
  if (grid <= 0) return 0;
  kern<<<grid, 32, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <int N, int M>
int launch_recon_t(const ReconArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(double) * RL<N, M>::TOTAL;
  const int64_t tasks = a.p.B * (int64_t)(a.seg_end - a.seg_begin);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, recon_small_kernel<N, M>, 32, smem);
  const int64_t cap = (int64_t)sms_count() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(tasks < cap ? tasks : cap);
  if (grid <= 0) return 0;
  recon_small_kernel<N, M><<<grid, 32, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <int N>
int launch_link_t(const plq_problem_t& p, const double* vf0, double* links, double* link_residual, int32_t* status,
                  double* ws, cudaStream_t s) {
  const int J = p.J, K = J - 1;
  const size_t smem = sizeof(double) * (3 * (size_t)(3 * N * N + 2 * N) + 3 * N * (N + 1) + K * N + N +
                                        (N * (N + 1) + 7) / 8 + 1 + 4);
  auto kern = link_seq_kernel<N>;
  static unsigned attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, smem);
  const int64_t cap = (int64_t)sms_count() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(p.B < cap ? p.B : cap);
  kern<<<grid, 32, smem, s>>>(p, vf0, links, link_residual, status, ws);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace

template <int N, int M, int NT, int RS>
int launch_recon_ring(const ReconArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(double) * ((size_t)RS * RingL<N, M>::SLOT + (N >= 64 ? 0 : 2 * N * N + 2 * N) +
                                        (size_t)a.p.max_seg_len * (N + M) + 10 * N + 6 * M + NT / 32 + 16);
  auto kern = recon_ring_kernel<N, M, NT, RS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
  const int64_t tasks = a.p.B * (int64_t)(a.seg_end - a.seg_begin);
  const int64_t cap = (int64_t)sms_count() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(tasks < cap ? tasks : cap);
  if (grid <= 0) return 0;
  kern<<<grid, NT, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

bool recon_small_supported(int n, int m) { return (n == 12 && m == 4) || (n == 32 && m == 8) || (n == 64 && m == 32); }

int launch_recon_small(const ReconArgs& a, cudaStream_t s) {
  // n = 32 / 64: forward rollout, stage-parallel evaluation and backward
  // multipliers as three streaming kernels (plq_recon_ring.cu); the fused
  // single-kernel ring (PLQ_RECON_FUSED=1) is kept for measurement
  const char* fused = getenv("PLQ_RECON_FUSED");
  if (recon_split_supported(a.p.n, a.p.m) && !(fused && fused[0] == '1')) return launch_recon_split(a, s);
  if (a.p.n == 64 && a.p.m == 32) {
    if (a.p.max_seg_len <= 128) return launch_recon_ring<64, 32, 256, 1>(a, s);
    return -1;
  }
  if (a.p.n == 32 && a.p.m == 8) {
    if (a.p.max_seg_len <= 512) return launch_recon_ring<32, 8, 128, 2>(a, s);  // 2 slots: 2 CTAs per SM
    return -1;
  }
  if (a.p.n == 12 && a.p.m == 4) {
    // whole segment on chip when it fits (BASELINE config 1: L = 8)
    if (a.p.max_seg_len <= 8) return launch_recon_seg<12, 4, 8>(a, s);
    return launch_recon_t<12, 4>(a, s);
  }
  return -1;
}

// the sequential link solve is used while the chain is short (J <= 64 at n = 12)
bool link_seq_supported(int n, int J) { return n == 12 && J <= 64; }

size_t link_seq_workspace_doubles(int64_t B, int J, int n) { return (size_t)B * (J - 1) * n * n + 2; }

int launch_link_seq(const plq_problem_t& p, const double* vf0, double* links, double* link_residual,
                    int32_t* status, double* ws, cudaStream_t s) {
  if (p.J < 2) return 0;
  if (p.n == 12) return launch_link_t<12>(p, vf0, links, link_residual, status, ws, s);
  return -1;
}

}  // namespace plq
