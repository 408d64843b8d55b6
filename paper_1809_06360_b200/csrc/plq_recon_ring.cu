// K3 for n >= 32 (BASELINE configs 2 and 4): the segment reconstruction of
// solve_parallel (parallel.py:478-527) split by what carries a recurrence.
//
//   recon_fwd_kernel   the rollout u_s = Kx x_s + (Kz z + k1), x_{s+1} = Fx x_s
//                      + Fu u_s + f1 (parallel.py:495-502): per stage only
//                      Fx, Fu, f1, Kx, Kz, k1 are streamed (TMA 1-D ring);
//   recon_eval_kernel  stage-parallel, no recurrence: the stationarity terms
//                      g = Qxx x + Qux' u + qx1, h = Qux x + Quu u + qu1 and the
//                      stage objective (problem.py:366-382);
//   recon_bwd_kernel   the multiplier recursion lambda_s = Fx' lambda_{s+1} - g
//                      (parallel.py:505-523) and the interior KKT rows, with
//                      Fx, Fu and g/h streamed.
//
// The single-kernel ring variant streamed all eleven stage fields (141 KB
// per stage at n = 64) through one slot, so every stage waited for its own
// copy; here the recurrent passes stream 83 / 50 KB per stage through 2- /
// 3-slot rings and the Q-block work runs at streaming bandwidth.
#include <stdlib.h>

#include "plq_device.cuh"
#include "plq_internal.h"
#include "plq_tma.cuh"

namespace plq {

namespace {

template <int N, int M>
struct FwdL {   // Fx | Fu | f1 | Kx | Kz | k1
  static constexpr int NN = N * N, NM = N * M;
  static constexpr int FX = 0, FU = NN, F1 = FU + NM, KX = F1 + N, KZ = KX + NM, K1 = KZ + NM;
  static constexpr int SLOT = (K1 + M + 1) & ~1;
  static constexpr uint32_t BYTES = 8u * (NN + 3 * NM + N + M);
};

template <int N, int M>
struct EvalL {  // Qxx | Qux | Quu | qx1 | qu1 | x | u
  static constexpr int NN = N * N, NM = N * M, MM = M * M;
  static constexpr int QXX = 0, QUX = NN, QUU = QUX + NM, QX1 = QUU + MM, QU1 = QX1 + N, X = QU1 + M, U = X + N;
  static constexpr int SLOT = (U + M + 1) & ~1;
  static constexpr uint32_t BYTES = 8u * (NN + NM + MM + 2 * N + 2 * M);
};

template <int N, int M>
struct BwdL {   // Fx | Fu | g h
  static constexpr int NN = N * N, NM = N * M;
  static constexpr int FX = 0, FU = NN, GH = FU + NM;
  static constexpr int SLOT = (GH + N + M + 1) & ~1;
  static constexpr uint32_t BYTES = 8u * (NN + NM + N + M);
};

template <int N, int M>
__device__ __forceinline__ void fwd_issue(const ReconArgs& A, double* slot, uint64_t* bar, int64_t st) {
  using R = FwdL<N, M>;
  fence_proxy_async();
  mbar_arrive_tx(bar, R::BYTES);
  bulk_g2s(slot + R::FX, A.p.Fx + st * R::NN, 8u * R::NN, bar);
  bulk_g2s(slot + R::FU, A.p.Fu + st * R::NM, 8u * R::NM, bar);
  bulk_g2s(slot + R::F1, A.p.f1 + st * N, 8u * N, bar);
  bulk_g2s(slot + R::KX, A.Kx + st * R::NM, 8u * R::NM, bar);
  bulk_g2s(slot + R::KZ, A.Kz + st * R::NM, 8u * R::NM, bar);
  bulk_g2s(slot + R::K1, A.k1 + st * M, 8u * M, bar);
}

template <int N, int M>
__device__ __forceinline__ void eval_issue(const ReconArgs& A, double* slot, uint64_t* bar, int64_t st, int64_t xrow) {
  using R = EvalL<N, M>;
  fence_proxy_async();
  mbar_arrive_tx(bar, R::BYTES);
  bulk_g2s(slot + R::QXX, A.p.Qxx + st * R::NN, 8u * R::NN, bar);
  bulk_g2s(slot + R::QUX, A.p.Qux + st * R::NM, 8u * R::NM, bar);
  bulk_g2s(slot + R::QUU, A.p.Quu + st * R::MM, 8u * R::MM, bar);
  bulk_g2s(slot + R::QX1, A.p.qx1 + st * N, 8u * N, bar);
  bulk_g2s(slot + R::QU1, A.p.qu1 + st * M, 8u * M, bar);
  bulk_g2s(slot + R::X, A.x + xrow * N, 8u * N, bar);
  bulk_g2s(slot + R::U, A.u + st * M, 8u * M, bar);
}

template <int N, int M>
__device__ __forceinline__ void bwd_issue(const ReconArgs& A, double* slot, uint64_t* bar, int64_t st) {
  using R = BwdL<N, M>;
  fence_proxy_async();
  mbar_arrive_tx(bar, R::BYTES);
  bulk_g2s(slot + R::FX, A.p.Fx + st * R::NN, 8u * R::NN, bar);
  bulk_g2s(slot + R::FU, A.p.Fu + st * R::NM, 8u * R::NM, bar);
  bulk_g2s(slot + R::GH, A.gh + st * (N + M), 8u * (N + M), bar);
}

// Row dot product with a per-lane rotated column order.  The bulk copies land
// the matrices unpadded, so the rows of consecutive lanes are K doubles apart
// and a plain rp[c] loop puts all 32 lanes of a load on the same bank (a
// 32-way conflict: ~6 k shared-memory wavefronts per n = 64 stage, more than
// the stage's HBM time).  Starting lane t at column pair (c + t) and loading
// 16 bytes spreads every quarter-warp over all eight 16-byte bank groups.
template <int K>
__device__ __forceinline__ double rdot_rot(const double* rp, const double* vec, int rot) {
  static_assert(K % 2 == 0 && ((K / 2) & (K / 2 - 1)) == 0, "row length: twice a power of two");
  const double2* r2 = reinterpret_cast<const double2*>(rp);
  const double2* v2 = reinterpret_cast<const double2*>(vec);
  double t = 0.0, t_ = 0.0;
#pragma unroll 8
  for (int c = 0; c < K / 2; ++c) {
    const int k = (c + rot) & (K / 2 - 1);
    const double2 a = r2[k], b = v2[k];
    t += a.x * b.x;
    t_ += a.y * b.y;
  }
  return t + t_;
}

template <int N, int M, int NT, int RS>
__global__ void __launch_bounds__(NT) recon_fwd_kernel(ReconArgs A) {
  using R = FwdL<N, M>;
  static_assert(N + 2 * M <= NT, "one thread per pass-1 row");
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = A.p;
  const int J = p.J, T = p.T, tid = threadIdx.x;
  double* ring = sm;
  double* x = ring + RS * R::SLOT;
  double* xn = x + N;
  double* z = xn + N;
  double* tf = z + N;
  double* uu = tf + N;
  double* tu = uu + M;
  double* tk = tu + M;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tk + M);
  if (tid == 0)
    for (int k = 0; k < RS; ++k) mbar_init(bars + k, 1);
  __syncthreads();
  uint32_t phases = 0u;   // bit k: parity of slot k's next completion
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t total = p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = A.seg_begin + (int)(task % nloc);
    const int lo = p.split_times[j], L = p.split_times[j + 1] - lo;
    if (!segment_bounds_ok(p, j)) continue;   // malformed partition (flagged by the sweep)
    const bool last = (j == J - 1);
    const int64_t s0 = b * T + lo;
    if (tid == 0)
      for (int k = 0; k < RS && k < L; ++k) fwd_issue<N, M>(A, ring + k * R::SLOT, bars + k, s0 + k);
    if (tid < N) {
      x[tid] = (j == 0) ? p.x_init[b * N + tid] : A.links[(b * (J - 1) + (j - 1)) * N + tid];
      z[tid] = last ? 0.0 : A.links[(b * (J - 1) + j) * N + tid];
    }
    __syncthreads();
#pragma unroll 1
    for (int s = 0; s < L; ++s) {
      const int slot = s % RS;
      const double* sl = ring + slot * R::SLOT;
      mbar_wait(bars + slot, (phases >> slot) & 1u);
      phases ^= 1u << slot;
      const int64_t st = s0 + s;
      // pass 1: Fx x | Kx x | Kz z
      if (tid < N)
        tf[tid] = rdot_rot<N>(sl + R::FX + tid * N, x, tid);
      else if (tid < N + M)
        tu[tid - N] = rdot_rot<N>(sl + R::KX + (tid - N) * N, x, tid);
      else if (tid < N + 2 * M)
        tk[tid - N - M] = rdot_rot<N>(sl + R::KZ + (tid - N - M) * N, z, tid);
      __syncthreads();
      if (tid < M) {
        const double kk = tk[tid] + sl[R::K1 + tid];   // k = Kz z + k1 (parallel.py:495)
        const double uv = tu[tid] + kk;
        uu[tid] = uv;
        A.k[st * M + tid] = kk;
        A.u[st * M + tid] = uv;
      } else if (tid >= NT - N) {
        const int i = tid - (NT - N);
        A.x[(b * (T + 1) + lo + s) * N + i] = x[i];
      }
      __syncthreads();
      if (tid < N) {
        const double t = rdot_rot<M>(sl + R::FU + tid * M, uu, tid);
        xn[tid] = (tf[tid] + t) + sl[R::F1 + tid];
      }
      __syncthreads();
      if (tid == 0 && s + RS < L) fwd_issue<N, M>(A, ring + slot * R::SLOT, bars + slot, st + RS);
      if (tid < N) x[tid] = xn[tid];
      __syncthreads();
    }
    if (tid < N) {
      if (last)
        A.x[(b * (T + 1) + T) * N + tid] = x[tid];
      else
        A.xend[(b * J + j) * N + tid] = x[tid];
    }
    __syncthreads();
  }
}

template <int N, int M, int NT, int RS>
__global__ void __launch_bounds__(NT) recon_eval_kernel(ReconArgs A) {
  using R = EvalL<N, M>;
  static_assert(N + M <= NT, "one thread per row");
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = A.p;
  const int J = p.J, T = p.T, tid = threadIdx.x;
  double* ring = sm;
  double* t0 = ring + RS * R::SLOT;   // Qxx x
  double* t2 = t0 + N;                // Qux x
  double* red = t2 + M;
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + NT / 32 + ((N + M + NT / 32) & 1));
  if (tid == 0)
    for (int k = 0; k < RS; ++k) mbar_init(bars + k, 1);
  __syncthreads();
  uint32_t phases = 0u;   // bit k: parity of slot k's next completion
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t total = p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = A.seg_begin + (int)(task % nloc);
    const int lo = p.split_times[j], L = p.split_times[j + 1] - lo;
    if (!segment_bounds_ok(p, j)) continue;   // malformed partition (flagged by the sweep)
    const int64_t s0 = b * T + lo, x0 = b * (T + 1) + lo;
    if (tid == 0)
      for (int k = 0; k < RS && k < L; ++k) eval_issue<N, M>(A, ring + k * R::SLOT, bars + k, s0 + k, x0 + k);
    double obj = 0.0;
#pragma unroll 1
    for (int s = 0; s < L; ++s) {
      const int slot = s % RS;
      const double* sl = ring + slot * R::SLOT;
      mbar_wait(bars + slot, (phases >> slot) & 1u);
      phases ^= 1u << slot;
      const int64_t st = s0 + s;
      if (tid < N)
        t0[tid] = rdot_rot<N>(sl + R::QXX + tid * N, sl + R::X, tid);
      else if (tid < N + M)
        t2[tid - N] = rdot_rot<N>(sl + R::QUX + (tid - N) * N, sl + R::X, tid);
      __syncthreads();
      if (tid < N) {
        // g = Qxx x + Qux' u + qx1; objective 1/2 x'Qxx x + qx1'x
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) t += sl[R::QUX + q * N + tid] * sl[R::U + q];
        const double xi = sl[R::X + tid], qx = sl[R::QX1 + tid];
        A.gh[st * (N + M) + tid] = (t0[tid] + t) + qx;
        obj += 0.5 * xi * t0[tid] + qx * xi;
      } else if (tid < N + M) {
        // h = Qux x + Quu u + qu1; objective 1/2 u'Quu u + u'Qux x + qu1'u
        const int u = tid - N;
        const double t = rdot_rot<M>(sl + R::QUU + u * M, sl + R::U, u);
        const double ui = sl[R::U + u], qu = sl[R::QU1 + u];
        A.gh[st * (N + M) + N + u] = (t2[u] + t) + qu;
        obj += 0.5 * ui * t + ui * t2[u] + qu * ui;
      }
      __syncthreads();
      if (tid == 0 && s + RS < L) eval_issue<N, M>(A, ring + slot * R::SLOT, bars + slot, st + RS, x0 + s + RS);
    }
    obj = block_sum(obj, red);
    if (tid == 0) A.part[(b * J + j) * 3 + 0] = obj;
    __syncthreads();
  }
}

template <int N, int M, int NT, int RS>
__global__ void __launch_bounds__(NT) recon_bwd_kernel(ReconArgs A) {
  using R = BwdL<N, M>;
  constexpr int NN = N * N;
  static_assert(N + M <= NT, "one thread per row");
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = A.p;
  const int J = p.J, T = p.T, tid = threadIdx.x;
  double* ring = sm;
  double* lam = ring + RS * R::SLOT;
  double* av = lam + N;
  double* z = av + N;
  double* red = z + N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + NT / 32 + ((3 * N + NT / 32) & 1));
  if (tid == 0)
    for (int k = 0; k < RS; ++k) mbar_init(bars + k, 1);
  __syncthreads();
  uint32_t phases = 0u;   // bit k: parity of slot k's next completion
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t total = p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = A.seg_begin + (int)(task % nloc);
    const int lo = p.split_times[j], L = p.split_times[j + 1] - lo;
    if (!segment_bounds_ok(p, j)) continue;   // malformed partition (flagged by the sweep)
    const bool last = (j == J - 1);
    const int64_t s0 = b * T + lo;
    if (tid == 0)
      for (int k = 0; k < RS && k < L; ++k) bwd_issue<N, M>(A, ring + k * R::SLOT, bars + k, s0 + L - 1 - k);
    if (tid < N) {
      // last segment: x_T; endpoint segment: its start point a and end point z
      av[tid] = last ? A.x[(b * (T + 1) + T) * N + tid]
                     : ((j == 0) ? p.x_init[b * N + tid] : A.links[(b * (J - 1) + (j - 1)) * N + tid]);
      z[tid] = last ? 0.0 : A.links[(b * (J - 1) + j) * N + tid];
    }
    __syncthreads();
    double obj = 0.0, worst = 0.0;
    // ---- multiplier seed (parallel.py:505-515)
    if (tid < N) {
      if (last) {
        // lambda_T = -(QxxT x_T + qx1T); terminal objective term
        double t = 0.0;
        const double* QT = p.QxxT + b * NN + tid * N;
        for (int c = 0; c < N; ++c) t += QT[c] * av[c];
        const double q1 = p.qx1T[b * N + tid], xT = av[tid];
        obj += 0.5 * xT * t + q1 * xT;
        const double g = t + q1;
        lam[tid] = -g;
        A.lam[(b * (T + 1) + T) * N + tid] = -g;
        worst = fmax(worst, fabs(g + -g));
      } else {
        // mu_j = -(Vzx0 a + Vzz0 z + vz10) (minus Hz'nu for degenerate segments)
        const double* vsrc = A.vf0 + (b * J + j) * (int64_t)(3 * NN + 2 * N) + NN;
        double t0v = 0.0, t1v = 0.0;
        for (int c = 0; c < N; ++c) {
          t0v += vsrc[tid * N + c] * av[c];
          t1v += vsrc[NN + tid * N + c] * z[c];
        }
        const double mu = -((t0v + t1v) + vsrc[2 * NN + N + tid]) -
                          (A.mu_corr && A.feas_rows[b * J + j] > 0 ? A.mu_corr[(b * J + j) * N + tid] : 0.0);
        A.mu_left[(b * (J - 1) + j) * N + tid] = mu;
        lam[tid] = -mu;
      }
    }
    __syncthreads();
    // ---- backward multipliers + interior KKT rows
#pragma unroll 1
    for (int k = 0; k < L; ++k) {
      const int s = L - 1 - k;
      const int slot = k % RS;
      const double* sl = ring + slot * R::SLOT;
      mbar_wait(bars + slot, (phases >> slot) & 1u);
      phases ^= 1u << slot;
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
        const double g = sl[R::GH + tid];
        ln = tb - g;
        A.lam[(b * (T + 1) + lo + s) * N + tid] = ln;
        if (interior) worst = fmax(worst, fabs((g + ln) - tb));
      } else if (tid < N + M && interior) {
        worst = fmax(worst, fabs(sl[R::GH + tid] - tb));
      }
      __syncthreads();
      if (tid == 0 && k + RS < L) bwd_issue<N, M>(A, ring + slot * R::SLOT, bars + slot, s0 + s - RS);
      if (tid < N) lam[tid] = ln;
      __syncthreads();
    }
    if (j > 0 && tid < N) A.lambda_right[(b * (J - 1) + (j - 1)) * N + tid] = lam[tid];
    worst = block_max(worst, red);
    if (last) obj = block_sum(obj, red);
    if (tid == 0) {
      A.part[(b * J + j) * 3 + 1] = worst;
      if (last) A.part[(b * J + j) * 3 + 0] += obj;   // after recon_eval_kernel (stream order)
    }
    __syncthreads();
  }
}

int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <class K>
int launch_persistent(K kern, int threads, size_t smem, int64_t tasks, const ReconArgs& a, cudaStream_t s) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  const int64_t cap = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(tasks < cap ? tasks : cap);
  if (grid <= 0) return 0;
  kern<<<grid, threads, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <int N, int M, int NT, int RSF, int RSE, int RSB>
int launch_split(const ReconArgs& a, cudaStream_t s) {
  const int64_t tasks = a.p.B * (int64_t)(a.seg_end - a.seg_begin);
  const size_t fsm = sizeof(double) * ((size_t)RSF * FwdL<N, M>::SLOT + 4 * N + 3 * M + 2) + 8 * RSF;
  const size_t esm = sizeof(double) * ((size_t)RSE * EvalL<N, M>::SLOT + N + M + NT / 32 + 2) + 8 * RSE;
  const size_t bsm = sizeof(double) * ((size_t)RSB * BwdL<N, M>::SLOT + 3 * N + NT / 32 + 2) + 8 * RSB;
  if (launch_persistent(recon_fwd_kernel<N, M, NT, RSF>, NT, fsm, tasks, a, s)) return -1;
  if (launch_persistent(recon_eval_kernel<N, M, NT, RSE>, NT, esm, tasks, a, s)) return -1;
  return launch_persistent(recon_bwd_kernel<N, M, NT, RSB>, NT, bsm, tasks, a, s);
}

}  // namespace

// n = 64 / m = 32 (cfg4) and n = 32 / m = 8 (cfg2)
bool recon_split_supported(int n, int m) { return (n == 64 && m == 32) || (n == 32 && m == 8); }

int launch_recon_split(const ReconArgs& a, cudaStream_t s) {
  // ring depths (fwd, eval, bwd).  n = 64: one slot per CTA and 2-4 CTAs per
  // SM beat deep rings in one CTA (cfg4 recon 15.3 -> 12.7 ms with (1,1,1)
  // vs (2,3,3)); PLQ_RECON_RS selects measurement variants.
  const char* e = getenv("PLQ_RECON_RS");
  const int v = (e && e[0] >= '0' && e[0] <= '9') ? e[0] - '0' : 0;
  if (a.p.n == 64 && a.p.m == 32) {
    if (v == 2) return launch_split<64, 32, 128, 1, 2, 2>(a, s);
    if (v == 3) return launch_split<64, 32, 128, 2, 3, 3>(a, s);
    return launch_split<64, 32, 128, 1, 1, 1>(a, s);
  }
  if (a.p.n == 32 && a.p.m == 8) {   // cfg2 recon 0.79 -> 0.57 ms with (2,2,2) vs (4,4,4)
    if (v == 1) return launch_split<32, 8, 64, 1, 1, 1>(a, s);
    if (v == 4) return launch_split<32, 8, 64, 4, 4, 4>(a, s);
    return launch_split<32, 8, 64, 2, 2, 2>(a, s);
  }
  return -1;
}

}  // namespace plq
