// K3/K4: reconstruction of x_t, u_t, k_t, lambda_t from the solved links,
// per-segment objective / KKT partials, link-stage KKT rows and the final
// fixed-order reductions.
//
// Restates parallel.solve_parallel's reconstruction loop
// (/root/reference/pkg/src/parlqr/parallel.py:478-527) per segment in
// parallel, plus evaluate_objective / stationarity_residuals / kkt_residual
// (problem.py:366-420).  Matrices are read straight from global memory in
// coalesced order (each is used once per direction), vectors live in smem.
#include "plq_device.cuh"
#include "plq_internal.h"

namespace plq {

namespace {

// y[i] = sum_k A[i][k] x[k] (+ add[i]) for an R x C row-major matrix in
// global memory; warp per row with lanes striding the columns (coalesced).
__device__ __forceinline__ void gemv_rows(int R, int C, const double* __restrict__ A, const double* x, double* y,
                                          const double* add, double sign = 1.0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // four rows per trip: their loads are independent, so one memory latency
  // covers four rows instead of one (the matrices stream from HBM / L2)
  for (int i0 = warp; i0 < R; i0 += 4 * nw) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = lane; k < C; k += 32) {
      const double xv = x[k];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = i0 + e * nw;
        s[e] += (i < R ? A[(int64_t)i * C + k] : 0.0) * xv;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = i0 + e * nw;
      const double t = warp_sum(s[e]);
      if (lane == 0 && i < R) y[i] = sign * t + (add ? add[i] : 0.0);
    }
  }
}

// y[i] = sum_k A[k][i] x[k] for an R x C row-major matrix (y has C entries);
// thread per output column, rows walked in order (coalesced across threads).
__device__ __forceinline__ void gemv_cols(int R, int C, const double* __restrict__ A, const double* x, double* y) {
  for (int i = threadIdx.x; i < C; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < R; ++k) s += A[(int64_t)k * C + i] * x[k];
    y[i] = s;
  }
}

// Same product with the rows split over the CTA when it has more threads
// than columns: blockDim / C chunks of rows, per-chunk partial sums in `part`
// (blockDim doubles), summed in chunk order (deterministic).  Ends with a
// barrier; all threads must call it.
__device__ __forceinline__ void gemv_cols_par(int R, int C, const double* __restrict__ A, const double* x,
                                              double* y, double* part) {
  const int S = blockDim.x / C;
  if (S < 2) {
    gemv_cols(R, C, A, x, y);
    __syncthreads();
    return;
  }
  const int tid = threadIdx.x, chunk = tid / C, i = tid % C;
  if (chunk < S) {
    const int r0 = (int)((int64_t)R * chunk / S), r1 = (int)((int64_t)R * (chunk + 1) / S);
    double t0 = 0.0, t1 = 0.0;
    int k = r0;
    // eight rows per trip, loads first: one memory latency per eight rows
    for (; k + 7 < r1; k += 8) {
      double av[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) av[e] = A[(int64_t)(k + e) * C + i];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        t0 += av[e] * x[k + e];
        t1 += av[e + 1] * x[k + e + 1];
      }
    }
    for (; k + 1 < r1; k += 2) {
      t0 += A[(int64_t)k * C + i] * x[k];
      t1 += A[(int64_t)(k + 1) * C + i] * x[k + 1];
    }
    if (k < r1) t0 += A[(int64_t)k * C + i] * x[k];
    part[chunk * C + i] = t0 + t1;
  }
  __syncthreads();
  for (int c = tid; c < C; c += blockDim.x) {
    double t = 0.0;
    for (int h = 0; h < S; ++h) t += part[h * C + c];
    y[c] = t;
  }
  __syncthreads();
}

struct ReconSmem {
  double *x, *xn, *u, *k, *lam, *t0, *t1, *t2, *t3, *z, *a, *red, *part;
};

template <int NT>
__global__ void __launch_bounds__(NT, (NT == 512 ? 2 : 1)) recon_kernel(ReconArgs A) {
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = A.p;
  const int n = p.n, m = p.m, J = p.J, T = p.T, nn = n * n;
  const int tid = threadIdx.x, nt = blockDim.x;
  ReconSmem s;
  s.x = sm;
  s.xn = s.x + n;
  s.lam = s.xn + n;
  s.t0 = s.lam + n;
  s.t1 = s.t0 + n;
  s.z = s.t1 + n;
  s.a = s.z + n;
  s.u = s.a + n;
  s.k = s.u + m;
  s.t2 = s.k + m;
  s.t3 = s.t2 + m;
  s.red = s.t3 + m;
  s.part = s.red + 32;   // blockDim doubles (gemv_cols_par)
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t total = p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = A.seg_begin + (int)(task % nloc);
    const int lo = p.split_times[j], hi = p.split_times[j + 1], L = hi - lo;
    if (!segment_bounds_ok(p, j)) continue;   // malformed partition (flagged by the sweep)
    const bool last = (j == J - 1);
    const int vsz = 3 * nn + 2 * n;
    const double* vf = A.vf0 + (b * J + j) * (int64_t)vsz;
    // boundary states: a = x_init or the left link, z = the right link
    for (int i = tid; i < n; i += nt) {
      s.a[i] = (j == 0) ? p.x_init[b * n + i] : A.links[(b * (J - 1) + (j - 1)) * n + i];
      s.z[i] = last ? 0.0 : A.links[(b * (J - 1) + j) * n + i];
      s.x[i] = s.a[i];
    }
    __syncthreads();
    double obj = 0.0, kkt = 0.0;
    // ---- forward: fold k = Kz z + k1, rollout u = Kx x + k, x' = Fx x + Fu u + f1
    for (int sidx = 0; sidx < L; ++sidx) {
      const int64_t st = b * T + lo + sidx;
      const double* Kx = A.Kx + st * m * n;
      const double* Qxx = p.Qxx + st * nn;
      const double* Qux = p.Qux + st * m * n;
      const double* Quu = p.Quu + st * m * m;
      const double* Fx = p.Fx + st * nn;
      const double* Fu = p.Fu + st * n * m;
      if (last) {
        for (int i = tid; i < m; i += nt) s.k[i] = A.k1[st * m + i];
      } else {
        gemv_rows(m, n, A.Kz + st * m * n, s.z, s.k, A.k1 + st * m);
      }
      __syncthreads();
      gemv_rows(m, n, Kx, s.x, s.u, s.k);
      __syncthreads();
      for (int i = tid; i < m; i += nt) {
        A.k[st * m + i] = s.k[i];
        A.u[st * m + i] = s.u[i];
      }
      for (int i = tid; i < n; i += nt) A.x[(b * (T + 1) + lo + sidx) * n + i] = s.x[i];
      // g = Qxx x + Qux' u + qx1 ; h = Qux x + Quu u + qu1 ; x' = Fx x + Fu u + f1
      gemv_rows(n, n, Qxx, s.x, s.t0, nullptr);          // Qxx x
      gemv_cols(m, n, Qux, s.u, s.t1);                    // Qux' u
      gemv_rows(m, n, Qux, s.x, s.t2, nullptr);           // Qux x
      gemv_rows(m, m, Quu, s.u, s.t3, nullptr);           // Quu u
      __syncthreads();
      // stage cost (problem.py:378-379)
      double part = 0.0;
      for (int i = tid; i < n; i += nt) part += 0.5 * s.x[i] * s.t0[i] + p.qx1[st * n + i] * s.x[i];
      for (int i = tid; i < m; i += nt) part += 0.5 * s.u[i] * s.t3[i] + s.u[i] * s.t2[i] + p.qu1[st * m + i] * s.u[i];
      obj += block_sum(part, s.red);
      double* gh = A.gh + st * (n + m);
      for (int i = tid; i < n; i += nt) gh[i] = (s.t0[i] + s.t1[i]) + p.qx1[st * n + i];
      for (int i = tid; i < m; i += nt) gh[n + i] = (s.t2[i] + s.t3[i]) + p.qu1[st * m + i];
      __syncthreads();
      gemv_rows(n, n, Fx, s.x, s.t0, nullptr);
      gemv_rows(n, m, Fu, s.u, s.t1, nullptr);
      __syncthreads();
      for (int i = tid; i < n; i += nt) s.xn[i] = (s.t0[i] + s.t1[i]) + p.f1[st * n + i];
      __syncthreads();
      for (int i = tid; i < n; i += nt) s.x[i] = s.xn[i];
      __syncthreads();
    }
    // ---- multiplier seed (parallel.py:505-515)
    if (last) {
      const double* QT = p.QxxT + b * nn;
      for (int i = tid; i < n; i += nt) A.x[(b * (T + 1) + T) * n + i] = s.x[i];
      gemv_rows(n, n, QT, s.x, s.t1, nullptr);            // QxxT xT
      __syncthreads();
      double part = 0.0;
      for (int i = tid; i < n; i += nt) {
        s.t0[i] = s.t1[i] + p.qx1T[b * n + i];
        part += 0.5 * s.x[i] * s.t1[i] + p.qx1T[b * n + i] * s.x[i];
      }
      obj += block_sum(part, s.red);
      double worst = 0.0;
      for (int i = tid; i < n; i += nt) {
        const double lamT = -s.t0[i];
        s.lam[i] = lamT;
        A.lam[(b * (T + 1) + T) * n + i] = lamT;
        worst = fmax(worst, fabs(s.t0[i] + lamT));    // terminal row (problem.py:400)
      }
      kkt = fmax(kkt, block_max(worst, s.red));
    } else {
      for (int i = tid; i < n; i += nt) A.xend[(b * J + j) * n + i] = s.x[i];
      // mu = -(Vzx0 a + Vzz0 z + vz10)
      gemv_rows(n, n, vf + nn, s.a, s.t0, nullptr);
      gemv_rows(n, n, vf + 2 * nn, s.z, s.t1, nullptr);
      __syncthreads();
      for (int i = tid; i < n; i += nt) {
        const double mu = -((s.t0[i] + s.t1[i]) + vf[3 * nn + n + i]) - (A.mu_corr && A.feas_rows[b * J + j] > 0 ? A.mu_corr[(b * J + j) * n + i] : 0.0);
        A.mu_left[(b * (J - 1) + j) * n + i] = mu;
        s.lam[i] = -mu;
      }
    }
    __syncthreads();
    // ---- backward multiplier recursion (parallel.py:518-523) + interior KKT rows
    double worst = 0.0;
    for (int sidx = L - 1; sidx >= 0; --sidx) {
      const int64_t st = b * T + lo + sidx;
      const double* Fx = p.Fx + st * nn;
      const double* Fu = p.Fu + st * n * m;
      const double* gh = A.gh + st * (n + m);
      gemv_cols_par(n, n, Fx, s.lam, s.t0, s.part);     // Fx' lam_next
      gemv_cols_par(n, m, Fu, s.lam, s.t2, s.part);     // Fu' lam_next
      const bool interior = last || (sidx < L - 1);
      for (int i = tid; i < n; i += nt) {
        const double g = gh[i];
        const double lnew = s.t0[i] - g;
        s.xn[i] = lnew;
        A.lam[(b * (T + 1) + lo + sidx) * n + i] = lnew;
        if (interior) worst = fmax(worst, fabs((g + lnew) - s.t0[i]));
      }
      if (interior)
        for (int i = tid; i < m; i += nt) worst = fmax(worst, fabs(gh[n + i] - s.t2[i]));
      __syncthreads();
      for (int i = tid; i < n; i += nt) s.lam[i] = s.xn[i];
      __syncthreads();
    }
    kkt = fmax(kkt, block_max(worst, s.red));
    if (j > 0)
      for (int i = tid; i < n; i += nt) A.lambda_right[(b * (J - 1) + (j - 1)) * n + i] = s.lam[i];
    if (tid == 0) {
      A.part[(b * J + j) * 3 + 0] = obj;
      A.part[(b * J + j) * 3 + 1] = kkt;
    }
    __syncthreads();
  }
}

// KKT rows of each link stage t = hi_j - 1 of an endpoint segment, which
// need the right neighbour's lambda (problem.py:396-399):
//   r1 = g + lam_t - Fx' lam_{t+1},  r2 = h - Fu' lam_{t+1},  r3 = z - rollout end.
template <int NT>
__global__ void __launch_bounds__(NT) boundary_kernel(ReconArgs A) {
  extern __shared__ __align__(16) double sm[];
  const plq_problem_t& p = A.p;
  const int n = p.n, m = p.m, J = p.J, T = p.T;
  const int tid = threadIdx.x;
  double* lamn = sm;
  double* t0 = lamn + n;
  double* t2 = t0 + n;
  double* red = t2 + m;
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t total = p.B * nloc;
  for (int64_t task = blockIdx.x; task < total; task += gridDim.x) {
    const int64_t b = task / nloc;
    const int j = A.seg_begin + (int)(task % nloc);
    if (j == J - 1) {
      if (tid == 0) A.part[(b * J + j) * 3 + 2] = 0.0;
      continue;
    }
    if (!segment_bounds_ok(p, j)) continue;
    const int hi = p.split_times[j + 1];
    const int64_t st = b * T + (hi - 1);
    for (int i = tid; i < n; i += blockDim.x) lamn[i] = A.lambda_right[(b * (J - 1) + j) * n + i];
    __syncthreads();
    gemv_cols(n, n, p.Fx + st * n * n, lamn, t0);
    gemv_cols(n, m, p.Fu + st * n * m, lamn, t2);
    __syncthreads();
    double worst = 0.0;
    const double* gh = A.gh + st * (n + m);
    for (int i = tid; i < n; i += blockDim.x) {
      const double lt = A.lam[(b * (T + 1) + hi - 1) * n + i];
      worst = fmax(worst, fabs((gh[i] + lt) - t0[i]));
      worst = fmax(worst, fabs(A.links[(b * (J - 1) + j) * n + i] - A.xend[(b * J + j) * n + i]));
    }
    for (int i = tid; i < m; i += blockDim.x) worst = fmax(worst, fabs(gh[n + i] - t2[i]));
    worst = block_max(worst, red);
    if (tid == 0) A.part[(b * J + j) * 3 + 2] = worst;
    __syncthreads();
  }
}

// Small states (n, m <= 16): one thread per link stage, so every link stage
// of the batch is in flight at once (the per-stage work is two tiny
// transposed mat-vecs; the CTA-per-stage form is launch/latency bound).
template <int N, int M>
__global__ void __launch_bounds__(128) boundary_small_kernel(ReconArgs A) {
  const plq_problem_t& p = A.p;
  const int J = p.J, T = p.T;
  const int nloc = A.seg_end - A.seg_begin;
  const int64_t task = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (task >= p.B * nloc) return;
  const int64_t b = task / nloc;
  const int j = A.seg_begin + (int)(task % nloc);
  if (j == J - 1) {
    A.part[(b * J + j) * 3 + 2] = 0.0;
    return;
  }
  if (!segment_bounds_ok(p, j)) return;
  const int hi = p.split_times[j + 1];
  const int64_t st = b * T + (hi - 1);
  double ln[N];
#pragma unroll
  for (int k = 0; k < N; ++k) ln[k] = A.lambda_right[(b * (J - 1) + j) * N + k];
  const double* Fx = p.Fx + st * N * N;
  const double* Fu = p.Fu + st * N * M;
  const double* gh = A.gh + st * (N + M);
  double worst = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double t0 = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) t0 += Fx[k * N + i] * ln[k];
    const double lt = A.lam[(b * (T + 1) + hi - 1) * N + i];
    worst = fmax(worst, fabs((gh[i] + lt) - t0));
    worst = fmax(worst, fabs(A.links[(b * (J - 1) + j) * N + i] - A.xend[(b * J + j) * N + i]));
  }
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double t2 = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) t2 += Fu[k * M + i] * ln[k];
    worst = fmax(worst, fabs(gh[N + i] - t2));
  }
  A.part[(b * J + j) * 3 + 2] = worst;
}

// objective = fixed-order sum of segment partials; kkt = max of all rows;
// link_mismatch = max |mu_left + lambda_right| (parallel.py:527).  The sum is
// deterministic: thread t adds a fixed contiguous run of segments, then a
// fixed butterfly / warp-order combine (independent of how segments were
// sharded across ranks).
__global__ void finalize_kernel(plq_problem_t p, const double* part, const double* mu_left, const double* lambda_right,
                                double* objective, double* kkt, double* mismatch) {
  __shared__ double red[32];
  const int64_t b = blockIdx.x;
  const int J = p.J, n = p.n, nt = blockDim.x, t = threadIdx.x;
  double worst = 0.0;
  for (int64_t idx = t; idx < (int64_t)(J - 1) * n; idx += nt)
    worst = fmax(worst, fabs(mu_left[b * (J - 1) * n + idx] + lambda_right[b * (J - 1) * n + idx]));
  worst = block_max(worst, red);
  const int per = (J + nt - 1) / nt;
  double obj = 0.0, kk = 0.0;
  for (int j = t * per; j < (t + 1) * per && j < J; ++j) {
    obj += part[(b * J + j) * 3 + 0];
    kk = fmax(kk, fmax(part[(b * J + j) * 3 + 1], part[(b * J + j) * 3 + 2]));
  }
  obj = block_sum(obj, red);
  kk = block_max(kk, red);
  if (t == 0) {
    objective[b] = obj;
    kkt[b] = kk;
    mismatch[b] = worst;
  }
}

int recon_threads(int n) {
  if (n <= 16) return 32;
  if (n <= 32) return 64;
  if (n <= 64) return 128;
  // n > 64 (cfg3: 256 segments, fewer than two per SM): the per-stage
  // matrix-vector products are latency bound, so spread their rows over
  // 16 warps
  return 512;
}

int grid_for(int64_t tasks, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t per_sm = (2048 / threads) < 32 ? (2048 / threads) : 32;   // resident-CTA limit
  const int64_t cap = (int64_t)sms * per_sm;
  return (int)(tasks < cap ? tasks : cap);
}

}  // namespace

int launch_recon(const ReconArgs& a, cudaStream_t s) {
  const int threads = recon_threads(a.p.n);
  const size_t smem = sizeof(double) * (7 * a.p.n + 4 * a.p.m + 40 + threads);
  const int64_t tasks = a.p.B * (a.seg_end - a.seg_begin);
  if (tasks <= 0) return 0;
  const int grid = grid_for(tasks, threads);
  switch (threads) {
    case 32:
      recon_kernel<32><<<grid, 32, smem, s>>>(a);
      break;
    case 64:
      recon_kernel<64><<<grid, 64, smem, s>>>(a);
      break;
    case 128:
      recon_kernel<128><<<grid, 128, smem, s>>>(a);
      break;
    default:
      recon_kernel<512><<<grid, 512, smem, s>>>(a);
      break;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_boundary(const ReconArgs& a, double* /*unused*/, cudaStream_t s) {
  const int threads = recon_threads(a.p.n);
  const size_t smem = sizeof(double) * (2 * a.p.n + a.p.m + 40);
  const int64_t tasks = a.p.B * (a.seg_end - a.seg_begin);
  if (tasks <= 0) return 0;
  if (a.p.n == 12 && a.p.m == 4) {
    boundary_small_kernel<12, 4><<<(unsigned)((tasks + 127) / 128), 128, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  const int grid = grid_for(tasks, threads);
  switch (threads) {
    case 32:
      boundary_kernel<32><<<grid, 32, smem, s>>>(a);
      break;
    case 64:
      boundary_kernel<64><<<grid, 64, smem, s>>>(a);
      break;
    default:
      boundary_kernel<128><<<grid, 128, smem, s>>>(a);
      break;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_finalize(const plq_problem_t& p, const double* part, const double* /*bpart*/, const double* mu_left,
                    const double* lambda_right, const double* /*link_res*/, double* objective, double* kkt,
                    double* mismatch, double* /*link_residual*/, cudaStream_t s) {
  finalize_kernel<<<(unsigned)p.B, p.J > 64 ? 1024 : 128, 0, s>>>(p, part, mu_left, lambda_right, objective, kkt,
                                                                   mismatch);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace plq
