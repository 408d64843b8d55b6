// Smoothing pass, part 2: rollout of the smoothed policies fused with the
// evaluation of the smoothed solution (parallel.py:556-633).
//
// Part 1 (the per-segment serial sweeps with conditioned terminal costs)
// reuses the sweep kernels through SweepArgs::smooth_vf0.  This kernel then
// walks each problem's horizon once, in order, as the reference does:
//
//   u_t = K_t x_t + k_t,  x_{t+1} = Fx_t x_t + Fu_t u_t + f1_t      (_rollout_policies, :556-564)
//
// with the parent solve's policies on the last segment (left unchanged by
// smooth(), :610-615), and fuses on the same pass
//   * evaluate_objective of the new trajectory (problem.py:366-382),
//   * kkt_residual against the PARENT multipliers (the smoothed solution
//     keeps result.lambdas, :619-629).  The dynamics row is identically zero
//     (the rollout computes x_{t+1} with the residual's own expression) and
//     so is the initial-state row, so only stationarity and terminal rows
//     are formed,
//   * smooth_deviation = max |x - x_parent|, |u - u_parent| (:616-617).
//
// The horizon is a true recurrence (x_{t+1} needs u_t needs x_t), so the
// parallelism is across problems: one CTA per problem, thread per row; the
// evaluation rows of stage t are computed off the critical path, and stage
// t+1's operands are touched (L1-prefetched) while stage t finishes.
#include <cuda_runtime.h>

#include "plq_device.cuh"
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

template <int NT>
__global__ void __launch_bounds__(NT) smooth_rollout_kernel(SmoothArgs a) {
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
      dev = fmax(dev, fabs(ui - a.u0[bt * m + i]));
      if (keep) {
        for (int c = 0; c < n; ++c) a.K[bt * nm + i * n + c] = Kt[i * n + c];
        a.k[bt * m + i] = kt[i];
      }
    }
    __syncthreads();
    const double* Fx = p.Fx + bt * nn;
    const double* Fu = p.Fu + bt * nm;
    const double* Qxx = p.Qxx + bt * nn;
    const double* Qux = p.Qux + bt * nm;
    const double* Quu = p.Quu + bt * (int64_t)m * m;
    const double* lam = a.lam0 + (b * (T + 1) + t) * n;
    const double* lamn = lam + n;
    // next state first (the recurrence), then this row's evaluation terms
    for (int i = tid; i < n; i += NT) {
      xn[i] = (dot4(Fx + i * n, 1, x, n) + dot4(Fu + i * m, 1, u, m)) + p.f1[bt * n + i];
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
    }
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
  // terminal cost and terminal stationarity row: QxxT x_T + qx1T + lambda_T
  const double* lamT = a.lam0 + (b * (T + 1) + T) * n;
  for (int i = tid; i < n; i += NT) {
    const double g = dot4(p.QxxT + b * nn + i * n, 1, x, n);
    const double qt = p.qx1T[b * n + i];
    obj += x[i] * (0.5 * g + qt);
    kkt = fmax(kkt, fabs(g + qt + lamT[i]));
  }
  const double o = block_sum(obj, red);
  const double kv = block_max(kkt, red);
  const double dv = block_max(dev, red);
  if (tid == 0) {
    a.objective[b] = o;
    a.kkt[b] = kv;
    a.deviation[b] = dv;
  }
}

}  // namespace

int launch_smooth_rollout(const SmoothArgs& a, cudaStream_t s) {
  const int w = a.p.n > a.p.m ? a.p.n : a.p.m;
  const size_t smem = sizeof(double) * (2 * a.p.n + a.p.m + 32);
  const dim3 grid((unsigned)a.p.B);
  if (w <= 32)
    smooth_rollout_kernel<32><<<grid, 32, smem, s>>>(a);
  else if (w <= 64)
    smooth_rollout_kernel<64><<<grid, 64, smem, s>>>(a);
  else
    smooth_rollout_kernel<128><<<grid, 128, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace plq
