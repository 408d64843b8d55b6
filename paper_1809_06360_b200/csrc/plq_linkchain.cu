// K2c: the link solve of MANY problems with short chains, one CTA per problem.
//
// The reference solves the SPD block-tridiagonal link system by sequential
// block Cholesky (LinkSystem.solve parallel.py:264-283 ->
// endpoint.solve_block_tridiagonal endpoint.py:410-438):
//   P_i = D_i - S_{i-1} X_{i-1},  X_i = P_i^{-1} S_i',  d_i = P_i^{-1} g_i,
//   x_i = d_i - X_i x_{i+1},
// with D_i = Vzz0_i + Vxx0_{i+1}, S_i = A(i+1,i) = Vzx0_{i+1},
// b_i = -vz1_i - vx1_{i+1} (- Vzx0_0 x_init for i = 0)  (parallel.py:286-319).
// Block cyclic reduction (plq_link.cu) trades ~2x the flops and ~4 log2(J)
// launches for sequential depth; with a batch of at least as many problems as
// chain blocks (cfg4: 256 problems x 31 blocks of n = 64) the batch already
// fills the GPU, so each problem runs the reference's own recurrence in one
// CTA: pivot block and right-hand sides in shared memory, blocked Cholesky
// with the forward solve fused (gchol8), Schur update as the Gram product
// W_S'W_S of W = L^{-1}[S_i' | g_i] on DMMA, X_i = L^{-T} W (gtrsm8), and a
// matvec-only back-substitution.  Two CTAs per SM overlap one problem's
// serial 8 x 8 diagonal factors with the other's DMMA phases.
#include "plq_blocked.cuh"
#include "plq_device.cuh"
#include "plq_internal.h"

namespace plq {

namespace {

constexpr int CHAIN_THREADS = 256;

__host__ __device__ inline int chain_ldl(int n) { return n + ((12 - n % 8) % 8); }             // = 4 (mod 8)
__host__ __device__ inline int chain_ldw(int n) { return ((n + 1 + 3) / 8) * 8 + 4; }          // >= n + 1, = 4 (mod 8)
__host__ __device__ inline size_t chain_smem_doubles(int n) {
  const int nbk = (n + 7) / 8;
  return (size_t)n * chain_ldl(n) + (size_t)n * chain_ldw(n) + (size_t)nbk * 64 + 8 * 64 + 4 * (size_t)n + 8;
}

// per problem: X_i (K n^2), d_i (K n), Gram scratch (n^2)
__host__ __device__ inline size_t chain_ws_per_problem(int K, int n) {
  return (size_t)K * n * n + (size_t)K * n + (size_t)n * n;
}

__global__ void __launch_bounds__(CHAIN_THREADS, 2)
    link_chain_kernel(plq_problem_t p, const double* __restrict__ vf0, double* links, double* link_residual,
                      int32_t* status, double* ws) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int flag;
  __shared__ double red[32];
  const int n = p.n, J = p.J, K = J - 1, w = n + 1;
  const int ldl = chain_ldl(n), ldw = chain_ldw(n), nbk = (n + 7) / 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nn = (int64_t)n * n, vs = 3 * nn + 2 * n;
  double* Pm = sm;                        // n x ldl  pivot block -> factor
  double* Wm = Pm + (size_t)n * ldl;      // n x ldw  [S_i' | g_i] -> W -> [X_i | d_i]
  double* Linv = Wm + (size_t)n * ldw;    // nbk x 64 diagonal-block inverses
  double* wsc = Linv + nbk * 64;          // 8 x 64   per-warp tiles
  double* gv = wsc + 8 * 64;              // n        S_{i} d_{i} (next right-hand-side correction)
  double* xa = gv + n;                    // n        x_{i+1} (back-substitution) / x_{i-1}
  double* xb = xa + n;                    // n        x_i
  double* xc = xb + n;                    // n        x_{i+1} (residual)
  auto csync = [] { __syncthreads(); };
  for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
    const double* v = vf0 + b * J * vs;
    double* Xg = ws + b * chain_ws_per_problem(K, n);
    double* dg = Xg + (size_t)K * nn;
    double* Gs = dg + (size_t)K * n;
    const double* xi = p.x_init + b * n;
    if (tid == 0) flag = 0;
    bool ok = true;
    for (int i = 0; i < K; ++i) {
      const double* left = v + (int64_t)i * vs;
      const double* right = left + vs;
      const bool has_r = i + 1 < K;
      // ---- assemble P_i = D_i - S_{i-1} X_{i-1} and [S_i' | g_i]
      // (four elements per thread and trip, all twelve / sixteen loads issued before the
      // stores: the value blocks stream from HBM / L2, one latency per trip)
      for (int idx0 = tid; idx0 < nn; idx0 += 4 * CHAIN_THREADS) {
        double vz[4], vx[4], gs[4], sv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t idx = idx0 + (int64_t)e * CHAIN_THREADS;
          const bool in = idx < nn;
          vz[e] = in ? left[2 * nn + idx] : 0.0;
          vx[e] = in ? right[idx] : 0.0;
          gs[e] = (in && i > 0) ? Gs[idx] : 0.0;
          sv[e] = (in && has_r) ? right[nn + idx] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int idx = idx0 + e * CHAIN_THREADS;
          if (idx < nn) {
            const int r = idx / n, c = idx % n;
            double pv = vz[e] + vx[e];
            if (i > 0) pv -= gs[e];
            Pm[r * ldl + c] = pv;
            // S_i' (r, c) = Vzx0_{i+1}[c][r]: read row-major (coalesced), store transposed
            Wm[c * ldw + r] = sv[e];
          }
        }
      }
      for (int r = tid; r < n; r += CHAIN_THREADS) {
        double g = -left[3 * nn + n + r] + -right[3 * nn + r];
        if (i == 0) {
          double t = 0.0;
          for (int c = 0; c < n; ++c) t += left[nn + r * n + c] * xi[c];
          g += -t;
        } else {
          g -= gv[r];
        }
        Wm[r * ldw + n] = g;
      }
      __syncthreads();
      // ---- L L' = P_i with W = L^{-1}[S_i' | g_i] fused in
      if (!gchol8<8>(Pm, n, ldl, Linv, &flag, tid, csync, nullptr, Wm, w, ldw, wsc)) {
        ok = false;
        break;
      }
      // ---- Schur terms of the next pivot: Gs = W_S'W_S, gv = W_S'W_b (= S_i X_i, S_i d_i)
      if (has_r) {
        cta_gemm<true, false, 2, 2>(n, w, n, Wm, ldw, Wm, ldw, [&](int r, int c, double acc) {
          if (c < n)
            Gs[r * n + c] = acc;
          else
            gv[r] = acc;
        });
      }
      __syncthreads();
      // ---- [X_i | d_i] = L^{-T} W
      gtrsm8<1, 8>(Pm, n, ldl, Linv, Wm, w, ldw, wsc, tid, csync);
      if (has_r)
        for (int idx = tid; idx < nn; idx += CHAIN_THREADS) Xg[(int64_t)i * nn + idx] = Wm[(idx / n) * ldw + idx % n];
      for (int r = tid; r < n; r += CHAIN_THREADS) dg[(int64_t)i * n + r] = Wm[r * ldw + n];
      __syncthreads();
    }
    double* x = links + b * (int64_t)K * n;
    if (!ok) {
      // LinkSingular (parallel.py:267-271): flagged; the links are zeroed
      if (tid == 0 && status[b * J] == 0) status[b * J] = PLQ_STATUS_LINK_SINGULAR;
      for (int idx = tid; idx < K * n; idx += CHAIN_THREADS) x[idx] = 0.0;
      if (tid == 0) link_residual[b] = 0.0;
      __syncthreads();
      continue;
    }
    // ---- back-substitution x_i = d_i - X_i x_{i+1} (warp per row, coalesced X rows)
    for (int r = tid; r < n; r += CHAIN_THREADS) {
      const double t = dg[(int64_t)(K - 1) * n + r];
      xa[r] = t;
      x[(int64_t)(K - 1) * n + r] = t;
    }
    __syncthreads();
    for (int i = K - 2; i >= 0; --i) {
      const double* Xi = Xg + (int64_t)i * nn;
      constexpr int NWP = CHAIN_THREADS / 32;
      for (int r0 = warp; r0 < n; r0 += 4 * NWP) {   // four rows per trip: one latency for four rows
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        for (int c = lane; c < n; c += 32) {
          const double xv = xa[c];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = r0 + e * NWP;
            t[e] += (r < n ? Xi[r * n + c] : 0.0) * xv;
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = r0 + e * NWP;
          const double ts = warp_sum(t[e]);
          if (lane == 0 && r < n) xb[r] = dg[(int64_t)i * n + r] - ts;
        }
      }
      __syncthreads();
      for (int r = tid; r < n; r += CHAIN_THREADS) {
        const double t = xb[r];
        xa[r] = t;
        x[(int64_t)i * n + r] = t;
      }
      __syncthreads();
    }
    // ---- residual of the assembled equations at the solved links (parallel.py:273-282)
    double worst = 0.0;
    for (int i = 0; i < K; ++i) {
      const double* left = v + (int64_t)i * vs;
      const double* right = left + vs;
      const bool has_l = i >= 1, has_r = i + 1 < K;
      for (int r = tid; r < n; r += CHAIN_THREADS) {
        xa[r] = has_l ? x[(int64_t)(i - 1) * n + r] : 0.0;
        xb[r] = x[(int64_t)i * n + r];
        xc[r] = has_r ? x[(int64_t)(i + 1) * n + r] : 0.0;
      }
      __syncthreads();
      // transposed term S_i' x_{i+1}: thread per output row r = column r of Vzx0_{i+1}
      for (int r = tid; r < n; r += CHAIN_THREADS) {
        double t = 0.0;
        if (has_r)
          for (int c = 0; c < n; ++c) t += right[nn + c * n + r] * xc[c];
        gv[r] = t;
      }
      __syncthreads();
      constexpr int NWP = CHAIN_THREADS / 32;
      for (int r0 = warp; r0 < n; r0 += 4 * NWP) {
        double tt[4] = {0.0, 0.0, 0.0, 0.0};
        for (int c = lane; c < n; c += 32) {
          double d0[4], d1[4], d2[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {   // loads of four rows first
            const int r = r0 + e * NWP;
            const bool in = r < n;
            d0[e] = in ? left[2 * nn + r * n + c] : 0.0;
            d1[e] = in ? right[r * n + c] : 0.0;
            d2[e] = (in && has_l) ? left[nn + r * n + c] : 0.0;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            tt[e] += (d0[e] + d1[e]) * xb[c];
            if (has_l) tt[e] += d2[e] * xa[c];
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
        const int r = r0 + e * NWP;
        const double t = warp_sum(tt[e]);
        if (lane == 0 && r < n) {
          double g = -left[3 * nn + n + r] + -right[3 * nn + r];
          if (i == 0) {
            double s = 0.0;
            for (int c = 0; c < n; ++c) s += left[nn + r * n + c] * xi[c];
            g += -s;
          }
          worst = fmax(worst, fabs(t + gv[r] - g));
        }
        }
      }
      __syncthreads();
    }
    worst = block_max(worst, red);
    if (tid == 0) link_residual[b] = worst;
    __syncthreads();
  }
}

}  // namespace

// the chain kernel serves blocks of 16 <= n <= 64 when the batch has at least
// as many problems as the chain has blocks (PLQ_LINK=chain forces it)
bool link_chain_supported(int n, int J) { return n >= 16 && n <= 64 && J >= 2; }
bool link_chain_preferred(int64_t B, int J) { return B >= 8 && B >= J - 1; }

size_t link_chain_workspace_doubles(int64_t B, int J, int n) {
  return (size_t)B * ((chain_ws_per_problem(J - 1, n) + 1) & ~size_t(1));
}

int launch_link_chain(const plq_problem_t& p, const double* vf0, double* links, double* link_residual,
                      int32_t* status, double* ws, cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = chain_smem_doubles(p.n) * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(link_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (int)(p.B < (int64_t)2 * sms ? p.B : 2 * sms);
  link_chain_kernel<<<grid, CHAIN_THREADS, smem, s>>>(p, vf0, links, link_residual, status, ws);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace plq
