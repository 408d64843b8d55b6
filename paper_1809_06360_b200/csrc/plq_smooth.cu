// Smoothing pass, part 2: rollout of the smoothed policies and evaluation of
// the smoothed solution (parallel.py:556-633).
//
// Part 1 (the per-segment serial sweeps with conditioned terminal costs)
// reuses the sweep kernels through SweepArgs::smooth_vf0.  Part 2 computes
//
//   u_t = K_t x_t + k_t,  x_{t+1} = Fx_t x_t + Fu_t u_t + f1_t      (_rollout_policies, :556-564)
//
// with the parent solve's policies on the last segment (left unchanged by
// smooth(), :610-615), and
//   * evaluate_objective of the new trajectory (problem.py:366-382),
//   * kkt_residual against the PARENT multipliers (the smoothed solution
//     keeps result.lambdas, :619-629): stationarity rows, terminal row,
//     dynamics rows (identically zero within a rollout, measured where
//     segment rollouts join), initial row (zero: x_0 = x_init is copied),
//   * smooth_deviation = max |x - x_parent|, |u - u_parent| (:616-617).
//
// Two schedules:
//   * many problems (B >= #SMs or J = 1): one CTA walks each problem's
//     horizon, evaluation fused into the walk (smooth_walk_kernel);
//   * few problems (the single-horizon configs): the horizon recurrence is
//     split at the partition.  K_map computes each segment's closed-loop
//     affine map x_hi = Phi_j x_lo + c_j by stepping [Phi | c] (n x (n+1))
//     through the segment on the FP64 tensor pipe; K_roll composes the maps
//     of the preceding segments into its start state and rolls the segment
//     out (recurrence only, stage operands double-buffered by cp.async);
//     K_eval evaluates objective / KKT / deviation stage-parallel; K_fin
//     reduces the partials in a fixed order.
#include <cuda_runtime.h>

#include <type_traits>

#include "plq_device.cuh"
#include "plq_gemm.cuh"
#include "plq_internal.h"

namespace plq {
namespace {

// Dot product with four independent accumulators (latency, not order, bound).
__device__ __forceinline__ double dot4(const double* __restrict__ a, int sa, const double* x, int len) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = 0;
  for (; k + 3 < len; k += 4) {
    s0 += a[(k + 0) * sa] * x[k + 0];
    s1 += a[(k + 1) * sa] * x[k + 1];
    s2 += a[(k + 2) * sa] * x[k + 2];
    s3 += a[(k + 3) * sa] * x[k + 3];
  }
  for (; k < len; ++k) s0 += a[k * sa] * x[k];
  return (s0 + s1) + (s2 + s3);
}

__device__ __forceinline__ void async_copy(double* dst, const double* src, int len) {
  for (int i = threadIdx.x; i < len; i += blockDim.x) cp_async8(dst + i, src + i, true);
}

// Evaluation rows of stage t given x_t, u_t (any memory), accumulated into
// this thread's objective sum and KKT / deviation maxima.
__device__ __forceinline__ void eval_stage(const SmoothArgs& a, int64_t b, int t, const double* x, const double* u,
                                           int NT, double& obj, double& kkt, double& dev) {
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, tid = threadIdx.x;
  const int64_t bt = b * T + t, nn = (int64_t)n * n, nm = (int64_t)n * m;
  const double* Fx = p.Fx + bt * nn;
  const double* Fu = p.Fu + bt * nm;
  const double* Qxx = p.Qxx + bt * nn;
  const double* Qux = p.Qux + bt * nm;
  const double* Quu = p.Quu + bt * (int64_t)m * m;
  const double* lam = a.lam0 + (b * (T + 1) + t) * n;
  const double* lamn = lam + n;
  for (int i = tid; i < n; i += NT) {
    const double g = dot4(Qxx + i * n, 1, x, n);
    const double qx = p.qx1[bt * n + i];
    const double r1 = g + dot4(Qux + i, n, u, m) + qx + lam[i] - dot4(Fx + i, n, lamn, n);
    kkt = fmax(kkt, fabs(r1));
    obj += x[i] * (0.5 * g + qx);
  }
  for (int i = tid; i < m; i += NT) {
    const double h = dot4(Qux + i * n, 1, x, n);
    const double hu = dot4(Quu + i * m, 1, u, m);
    const double qu = p.qu1[bt * m + i];
    const double r2 = h + hu + qu - dot4(Fu + i, m, lamn, n);
    kkt = fmax(kkt, fabs(r2));
    obj += u[i] * (0.5 * hu + h + qu);
    dev = fmax(dev, fabs(u[i] - a.u0[bt * m + i]));
  }
}

// Terminal cost and terminal stationarity row QxxT x_T + qx1T + lambda_T.
__device__ __forceinline__ void eval_terminal(const SmoothArgs& a, int64_t b, const double* x, int NT, double& obj,
                                              double& kkt) {
  const plq_problem_t& p = a.p;
  const int n = p.n, T = p.T;
  const double* lamT = a.lam0 + (b * (T + 1) + T) * n;
  for (int i = threadIdx.x; i < n; i += NT) {
    const double g = dot4(p.QxxT + b * (int64_t)n * n + i * n, 1, x, n);
    const double qt = p.qx1T[b * n + i];
    obj += x[i] * (0.5 * g + qt);
    kkt = fmax(kkt, fabs(g + qt + lamT[i]));
  }
}

// ---------------------------------------------------------------------------
// many problems: one CTA per problem, evaluation fused into the walk
template <int NT>
__global__ void __launch_bounds__(NT) smooth_walk_kernel(SmoothArgs a) {
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  const int64_t nn = (int64_t)n * n, nm = (int64_t)n * m;
  double* x = sm;
  double* xn = x + n;
  double* u = xn + n;
  double* red = u + m;
  const int tlast = p.split_times[p.J - 1];

  double obj = 0.0, kkt = 0.0, dev = 0.0;
  for (int i = tid; i < n; i += NT) {
    const double v = p.x_init[b * n + i];
    x[i] = v;
    a.x[b * (T + 1) * n + i] = v;
    dev = fmax(dev, fabs(v - a.x0[b * (T + 1) * n + i]));
  }
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    const int64_t bt = b * T + t;
    const bool keep = t >= tlast;   // last segment: parent policies
    const double* Kt = (keep ? a.K0 : a.K) + bt * nm;
    const double* kt = (keep ? a.k0 : a.k) + bt * m;
    for (int i = tid; i < m; i += NT) {
      const double ui = dot4(Kt + i * n, 1, x, n) + kt[i];
      u[i] = ui;
      a.u[bt * m + i] = ui;
      if (keep) {
        for (int c = 0; c < n; ++c) a.K[bt * nm + i * n + c] = Kt[i * n + c];
        a.k[bt * m + i] = kt[i];
      }
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT)
      xn[i] = (dot4(p.Fx + bt * nn + i * n, 1, x, n) + dot4(p.Fu + bt * nm + i * m, 1, u, m)) + p.f1[bt * n + i];
    eval_stage(a, b, t, x, u, NT, obj, kkt, dev);
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      const double v = xn[i];
      x[i] = v;
      a.x[(b * (T + 1) + t + 1) * n + i] = v;
      dev = fmax(dev, fabs(v - a.x0[(b * (T + 1) + t + 1) * n + i]));
    }
    // warm L1 with the next stage's policy row while the barrier drains
    if (t + 1 < T && tid < m) {
      const double* Kn = ((t + 1 >= tlast) ? a.K0 : a.K) + (bt + 1) * nm + tid * n;
      asm volatile("prefetch.global.L1 [%0];" ::"l"(Kn));
    }
    __syncthreads();
  }
  eval_terminal(a, b, x, NT, obj, kkt);
  const double o = block_sum(obj, red);
  const double kv = block_max(kkt, red);
  const double dv = block_max(dev, red);
  if (tid == 0) {
    a.objective[b] = o;
    a.kkt[b] = kv;
    a.deviation[b] = dv;
  }
}

// ---------------------------------------------------------------------------
// few problems: segment maps, segment rollouts, stage-parallel evaluation

struct MapLayout {
  int ldx;          // row stride of X / X2 / U (n+1 padded)
  int onchip;       // X / X2 / U in shared memory (else a per-CTA workspace slice)
  int staged;       // stage operands double-buffered in smem
  int K, k, Fx, Fu, f1, per;   // offsets within one stage buffer, buffer size
};

MapLayout map_layout(int n, int m) {
  MapLayout L{};
  L.ldx = n + 1 + ((n + 1) % 2);
  int o = 0;
  L.K = o;  o += m * n;
  L.k = o;  o += m;
  L.Fx = o; o += n * n;
  L.Fu = o; o += n * m;
  L.f1 = o; o += n;
  L.per = (o + 1) & ~1;
  const size_t base = sizeof(double) * (size_t)(2 * n + m) * L.ldx;
  L.onchip = base <= 200 * 1024;
  L.staged = L.onchip && base + sizeof(double) * 2 * (size_t)L.per <= 200 * 1024;
  return L;
}

size_t map_smem(int n, int m) {
  const MapLayout L = map_layout(n, m);
  return sizeof(double) * ((L.onchip ? (size_t)(2 * n + m) * L.ldx : 0) + (L.staged ? 2 * (size_t)L.per : 0));
}

// [Phi | c] of segment j < J-1: X <- Fx X + Fu (K X + [0 | k]) + [0 | f1]
// over the segment's stages, X_0 = [I | 0].
template <int NT>
__global__ void __launch_bounds__(NT) smooth_map_kernel(SmoothArgs a, MapLayout L, double* scratch) {
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, J = p.J, tid = threadIdx.x, ld = L.ldx;
  const int64_t b = blockIdx.x / (J - 1);
  const int j = (int)(blockIdx.x % (J - 1));
  const int lo = p.split_times[j], hi = p.split_times[j + 1];
  if (!segment_bounds_ok(p, j)) return;
  const int64_t nn = (int64_t)n * n, nm = (int64_t)n * m;
  double* X = L.onchip ? sm : scratch + (int64_t)blockIdx.x * (2 * n + m) * ld;
  double* X2 = X + n * ld;
  double* U = X2 + n * ld;
  double* buf = sm + (L.onchip ? (2 * n + m) * ld : 0);
  for (int idx = tid; idx < n * ld; idx += NT) X[idx] = ((idx / ld) == (idx % ld)) ? 1.0 : 0.0;
  auto issue = [&](int t, double* dst) {
    const int64_t bt = b * T + t;
    async_copy(dst + L.K, a.K + bt * nm, (int)nm);
    async_copy(dst + L.k, a.k + bt * m, m);
    async_copy(dst + L.Fx, p.Fx + bt * nn, (int)nn);
    async_copy(dst + L.Fu, p.Fu + bt * nm, (int)nm);
    async_copy(dst + L.f1, p.f1 + bt * n, n);
    cp_async_commit();
  };
  if (L.staged) issue(lo, buf);
  __syncthreads();
  for (int t = lo; t < hi; ++t) {
    const int64_t bt = b * T + t;
    const double *Kt, *kt, *Fx, *Fu, *f1;
    if (L.staged) {
      double* cur = buf + ((t - lo) & 1) * L.per;
      if (t + 1 < hi) {
        issue(t + 1, buf + ((t + 1 - lo) & 1) * L.per);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      Kt = cur + L.K; kt = cur + L.k; Fx = cur + L.Fx; Fu = cur + L.Fu; f1 = cur + L.f1;
    } else {
      Kt = a.K + bt * nm; kt = a.k + bt * m; Fx = p.Fx + bt * nn; Fu = p.Fu + bt * nm; f1 = p.f1 + bt * n;
    }
    cta_gemm<false, false, 1, 1>(m, n + 1, n, Kt, n, X, ld, [&](int i, int c, double v) {
      U[i * ld + c] = v + (c == n ? kt[i] : 0.0);
    });
    __syncthreads();
    cta_gemm<false, false, 1, 1>(n, n + 1, n, Fx, n, X, ld, [&](int i, int c, double v) {
      X2[i * ld + c] = v + (c == n ? f1[i] : 0.0);
    });
    __syncthreads();
    cta_gemm<false, false, 1, 1>(n, n + 1, m, Fu, m, U, ld, [&](int i, int c, double v) { X2[i * ld + c] += v; });
    __syncthreads();
    double* tmp = X;
    X = X2;
    X2 = tmp;
  }
  double* dst = a.maps + (b * (J - 1) + j) * nn + (b * (J - 1) + j) * n;   // (B,J-1,n,n+1)
  for (int idx = tid; idx < n * (n + 1); idx += NT) dst[idx] = X[(idx / (n + 1)) * ld + idx % (n + 1)];
}

struct RollLayout {
  int staged;
  int K, k, Fx, Fu, f1, per;
};

RollLayout roll_layout(int n, int m) {
  RollLayout L{};
  int o = 0;
  L.K = o;  o += m * n;
  L.k = o;  o += m;
  L.Fx = o; o += n * n;
  L.Fu = o; o += n * m;
  L.f1 = o; o += n;
  L.per = (o + 1) & ~1;
  L.staged = sizeof(double) * (2 * (size_t)L.per + 3 * n + m + 32) <= 200 * 1024;
  return L;
}

// Rollout of segment j from the start state composed through the maps of
// segments 0..j-1; the join residual |Phi_j x_lo + c_j - x_hi| is recorded.
template <int NT>
__global__ void __launch_bounds__(NT) smooth_roll_kernel(SmoothArgs a, RollLayout L, double* joins) {
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, T = p.T, J = p.J, tid = threadIdx.x;
  const int64_t b = blockIdx.x / J;
  const int j = (int)(blockIdx.x % J);
  const int lo = p.split_times[j], hi = p.split_times[j + 1];
  if (!segment_bounds_ok(p, j)) return;
  const int tlast = p.split_times[J - 1];
  const int64_t nn = (int64_t)n * n, nm = (int64_t)n * m;
  double* x = sm;
  double* xn = x + n;
  double* xs = xn + n;
  double* u = xs + n;
  double* red = u + m;
  double* buf = red + 32;
  const double* maps = a.maps + b * (J - 1) * (nn + n);
  for (int i = tid; i < n; i += NT) x[i] = p.x_init[b * n + i];
  __syncthreads();
  for (int jj = 0; jj < j; ++jj) {   // x_lo = (maps of segments 0..j-1) x_init
    const double* Mj = maps + jj * (nn + n);
    for (int i = tid; i < n; i += NT) xn[i] = dot4(Mj + i * (n + 1), 1, x, n) + Mj[i * (n + 1) + n];
    __syncthreads();
    for (int i = tid; i < n; i += NT) x[i] = xn[i];
    __syncthreads();
  }
  for (int i = tid; i < n; i += NT) {
    xs[i] = x[i];
    a.x[(b * (T + 1) + lo) * n + i] = x[i];
  }
  auto issue = [&](int t, double* dst) {
    const int64_t bt = b * T + t;
    const bool keep = t >= tlast;
    async_copy(dst + L.K, (keep ? a.K0 : a.K) + bt * nm, (int)nm);
    async_copy(dst + L.k, (keep ? a.k0 : a.k) + bt * m, m);
    async_copy(dst + L.Fx, p.Fx + bt * nn, (int)nn);
    async_copy(dst + L.Fu, p.Fu + bt * nm, (int)nm);
    async_copy(dst + L.f1, p.f1 + bt * n, n);
    cp_async_commit();
  };
  if (L.staged) issue(lo, buf);
  __syncthreads();
  for (int t = lo; t < hi; ++t) {
    const int64_t bt = b * T + t;
    const bool keep = t >= tlast;
    const double *Kt, *kt, *Fx, *Fu, *f1;
    if (L.staged) {
      double* cur = buf + ((t - lo) & 1) * L.per;
      if (t + 1 < hi) {
        issue(t + 1, buf + ((t + 1 - lo) & 1) * L.per);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      Kt = cur + L.K; kt = cur + L.k; Fx = cur + L.Fx; Fu = cur + L.Fu; f1 = cur + L.f1;
    } else {
      Kt = (keep ? a.K0 : a.K) + bt * nm; kt = (keep ? a.k0 : a.k) + bt * m;
      Fx = p.Fx + bt * nn; Fu = p.Fu + bt * nm; f1 = p.f1 + bt * n;
    }
    for (int i = tid; i < m; i += NT) {
      const double ui = dot4(Kt + i * n, 1, x, n) + kt[i];
      u[i] = ui;
      a.u[bt * m + i] = ui;
      if (keep) {
        for (int c = 0; c < n; ++c) a.K[bt * nm + i * n + c] = Kt[i * n + c];
        a.k[bt * m + i] = kt[i];
      }
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT) xn[i] = (dot4(Fx + i * n, 1, x, n) + dot4(Fu + i * m, 1, u, m)) + f1[i];
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      x[i] = xn[i];
      if (t + 1 < hi || hi == T) a.x[(b * (T + 1) + t + 1) * n + i] = xn[i];
    }
    __syncthreads();
  }
  // dynamics row where this rollout meets the next segment's composed start
  double r3 = 0.0;
  if (j < J - 1) {
    const double* Mj = maps + j * (nn + n);
    for (int i = tid; i < n; i += NT)
      r3 = fmax(r3, fabs(dot4(Mj + i * (n + 1), 1, xs, n) + Mj[i * (n + 1) + n] - x[i]));
  }
  r3 = block_max(r3, red);
  if (tid == 0) joins[b * J + j] = r3;
}

// Stage-parallel evaluation: CTA per (problem, chunk of CH stages).
template <int NT>
__global__ void __launch_bounds__(NT) smooth_eval_kernel(SmoothArgs a, double* part, int nch) {
  __shared__ double red[32];
  const plq_problem_t& p = a.p;
  const int n = p.n, T = p.T, tid = threadIdx.x;
  const int64_t b = blockIdx.x / nch;
  const int c = (int)(blockIdx.x % nch);
  const int t0 = c * SMOOTH_EVAL_CH, t1 = min(T, t0 + SMOOTH_EVAL_CH);
  double obj = 0.0, kkt = 0.0, dev = 0.0;
  for (int t = t0; t < t1; ++t) {
    const double* x = a.x + (b * (T + 1) + t) * n;
    eval_stage(a, b, t, x, a.u + (b * T + t) * p.m, NT, obj, kkt, dev);
    for (int i = tid; i < n; i += NT) dev = fmax(dev, fabs(x[i] - a.x0[(b * (T + 1) + t) * n + i]));
  }
  if (t1 == T) {
    const double* x = a.x + (b * (T + 1) + T) * n;
    eval_terminal(a, b, x, NT, obj, kkt);
    for (int i = tid; i < n; i += NT) dev = fmax(dev, fabs(x[i] - a.x0[(b * (T + 1) + T) * n + i]));
  }
  const double o = block_sum(obj, red);
  const double kv = block_max(kkt, red);
  const double dv = block_max(dev, red);
  if (tid == 0) {
    double* q = part + (b * nch + c) * 3;
    q[0] = o;
    q[1] = kv;
    q[2] = dv;
  }
}

// Fixed-order reduction of the evaluation partials and join residuals.
__global__ void smooth_finalize_kernel(SmoothArgs a, const double* part, const double* joins, int nch) {
  __shared__ double red[32];
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, NT = blockDim.x, J = a.p.J;
  double kkt = 0.0, dev = 0.0;
  for (int c = tid; c < nch; c += NT) {
    kkt = fmax(kkt, part[(b * nch + c) * 3 + 1]);
    dev = fmax(dev, part[(b * nch + c) * 3 + 2]);
  }
  for (int j = tid; j < J; j += NT) kkt = fmax(kkt, joins[b * J + j]);
  // objective: per-thread contiguous chunks, then the block sum (fixed order)
  const int per = (nch + NT - 1) / NT;
  double obj = 0.0;
  for (int c = tid * per; c < min(nch, (tid + 1) * per); ++c) obj += part[(b * nch + c) * 3];
  const double o = block_sum(obj, red);
  const double kv = block_max(kkt, red);
  const double dv = block_max(dev, red);
  if (tid == 0) {
    a.objective[b] = o;
    a.kkt[b] = kv;
    a.deviation[b] = dv;
  }
}

template <class F>
int dispatch_nt(int w, F f) {
  if (w <= 32) return f(std::integral_constant<int, 32>());
  if (w <= 64) return f(std::integral_constant<int, 64>());
  return f(std::integral_constant<int, 128>());
}

}  // namespace

bool smooth_segmented(int64_t B, int J) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return J > 1 && B < (int64_t)sms;
}

size_t smooth_map_doubles(int64_t B, int T, int J, int n, int m) {
  const int nch = (T + SMOOTH_EVAL_CH - 1) / SMOOTH_EVAL_CH;
  const MapLayout L = map_layout(n, m);
  const size_t scratch = L.onchip ? 0 : (size_t)B * (J - 1) * (2 * n + m) * L.ldx;
  return (size_t)B * (J - 1) * n * (n + 1) + (size_t)B * J + (size_t)B * nch * 3 + scratch;
}

int launch_smooth_rollout(const SmoothArgs& a, cudaStream_t s, int* launches) {
  const plq_problem_t& p = a.p;
  const int n = p.n, m = p.m, J = p.J;
  const int w = n > m ? n : m;
  if (!smooth_segmented(p.B, J)) {
    const size_t smem = sizeof(double) * (2 * n + m + 32);
    *launches = 1;
    return dispatch_nt(w, [&](auto nt) {
      constexpr int NT = decltype(nt)::value;
      smooth_walk_kernel<NT><<<(unsigned)p.B, NT, smem, s>>>(a);
      return cudaGetLastError() == cudaSuccess ? 0 : -1;
    });
  }
  const int nch = (p.T + SMOOTH_EVAL_CH - 1) / SMOOTH_EVAL_CH;
  double* joins = a.maps + (size_t)p.B * (J - 1) * n * (n + 1);
  double* part = joins + (size_t)p.B * J;
  double* scratch = part + (size_t)p.B * nch * 3;
  // K_map: 128 threads (4 warps of DMMA tiles)
  {
    const MapLayout L = map_layout(n, m);
    const size_t smem = map_smem(n, m);
    auto kern = smooth_map_kernel<128>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
    kern<<<(unsigned)(p.B * (J - 1)), 128, smem, s>>>(a, L, scratch);
    if (cudaGetLastError() != cudaSuccess) return -1;
  }
  int rc = dispatch_nt(w, [&](auto nt) {
    constexpr int NT = decltype(nt)::value;
    const RollLayout L = roll_layout(n, m);
    const size_t smem = sizeof(double) * (3 * n + m + 32 + (L.staged ? 2 * (size_t)L.per : 0));
    auto kern = smooth_roll_kernel<NT>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
    kern<<<(unsigned)(p.B * J), NT, smem, s>>>(a, L, joins);
    if (cudaGetLastError() != cudaSuccess) return -1;
    smooth_eval_kernel<NT><<<(unsigned)(p.B * nch), NT, 0, s>>>(a, part, nch);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  });
  if (rc) return rc;
  smooth_finalize_kernel<<<(unsigned)p.B, 256, 0, s>>>(a, part, joins, nch);
  *launches = 4;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace plq
