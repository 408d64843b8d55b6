// K1 specialized: segment sweeps for the small-state configs (compile-time
// n, m; BASELINE configs 0-2: n=12/m=4 and n=32/m=8).
//
// Same recurrences as the generic sweep (plq_sweep.cu; endpoint.py:168-301,
// serial.py:37-79), restructured for latency:
//   * one group of NWG warps per segment, group barriers only;
//   * every buffer in shared memory with strides = 4 (mod 8) doubles so the
//     DMMA fragment loads are bank-conflict free;
//   * GEMM epilogues write in place: GEMM1 puts Mzx straight into Vzx (band
//     by band -- a band only reads its own rows) and Mzu' into P, GEMM2 puts
//     Mxx/mx1 into Vxx/vx1, and the value update accumulates into V;
//   * the next stage's inputs are loaded into registers while the current
//     stage computes (software pipelining over the stage loop).
#include "plq_internal.h"
#include "plq_small.cuh"

namespace plq {

namespace {

template <int N, int M>
struct SL {
  static constexpr int NN = N * N;
  static constexpr int LDN = pad_ld(N);
  static constexpr int FW = N + M + 1;
  static constexpr int LDF = pad_ld(FW);
  static constexpr int WE = 2 * N + 1;
  static constexpr int LDW = pad_ld(WE);
  static constexpr int SE = 2 * NN + 2 * N * M + M * M + 2 * N + M;   // stage input doubles
  static constexpr int V = 0;                    // Vxx, Vzx, Vzz: 3 x (N x LDN)
  static constexpr int VX1 = V + 3 * N * LDN;
  static constexpr int VZ1 = VX1 + N;
  static constexpr int F = (VZ1 + N + 1) & ~1;   // [Fx | Fu | f1]  N x LDF
  static constexpr int QXX = F + N * LDF;        // flat N x N
  static constexpr int QUX = QXX + NN;           // M x N
  static constexpr int QUU = QUX + M * N;        // M x M
  static constexpr int QX1 = QUU + M * M;        // N
  static constexpr int QU1 = QX1 + N;            // M
  static constexpr int VF = (QU1 + M + 1) & ~1;  // N x LDF (also N = Hx F)
  static constexpr int P = VF + N * LDF;         // P, G, Y: M x LDW each, contiguous
  static constexpr int G = P + M * LDW;
  static constexpr int Y = G + M * LDW;
  static constexpr int MUU = Y + M * LDW;        // M x M
  static constexpr int LM = MUU + M * M;         // M x M Cholesky factor
  static constexpr int IDG = LM + M * M;         // M   1 / L_ii
  static constexpr int H = IDG + M;              // N x LDW constraint rows [Hx | Hz | h1]
  static constexpr int TAU = H + N * LDW;        // M
  static constexpr int RD = TAU + M;             // M
  static constexpr int RED = RD + M;             // 8
  static constexpr int FLG = RED + 8;            // ints
  static constexpr int TOTAL = (FLG + 2 + 1) & ~1;
};

// stage element e (concatenation Fx|Fu|f1|Qxx|Qux|Quu|qx1|qu1) -> source
// address in global memory and destination offset in the group's smem
template <int N, int M>
__device__ __forceinline__ const double* stage_elem(const plq_problem_t& p, int64_t st, int e, int& dst) {
  using S = SL<N, M>;
  constexpr int NN = N * N, NM = N * M;
  if (e < NN) {
    dst = S::F + (e / N) * S::LDF + e % N;
    return p.Fx + st * NN + e;
  }
  e -= NN;
  if (e < NM) {
    dst = S::F + (e / M) * S::LDF + N + e % M;
    return p.Fu + st * NM + e;
  }
  e -= NM;
  if (e < N) {
    dst = S::F + e * S::LDF + N + M;
    return p.f1 + st * N + e;
  }
  e -= N;
  if (e < NN) {
    dst = S::QXX + e;
    return p.Qxx + st * NN + e;
  }
  e -= NN;
  if (e < NM) {
    dst = S::QUX + e;
    return p.Qux + st * NM + e;
  }
  e -= NM;
  if (e < M * M) {
    dst = S::QUU + e;
    return p.Quu + st * (M * M) + e;
  }
  e -= M * M;
  if (e < N) {
    dst = S::QX1 + e;
    return p.qx1 + st * N + e;
  }
  e -= N;
  dst = S::QU1 + e;
  return p.qu1 + st * M + e;
}

template <int N, int M, int NWG>
struct Prefetch {
  static constexpr int NT = NWG * 32;
  static constexpr int PF = (SL<N, M>::SE + NT - 1) / NT;
  double v[PF];
  __device__ __forceinline__ void load(const plq_problem_t& p, int64_t st, int gt) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int e = gt + k * NT;
      if (e < SL<N, M>::SE) {
        int d;
        v[k] = __ldg(stage_elem<N, M>(p, st, e, d));
      }
    }
  }
  __device__ __forceinline__ void store(const plq_problem_t& p, double* sm, int gt) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int e = gt + k * NT;
      if (e < SL<N, M>::SE) {
        int d;
        stage_elem<N, M>(p, 0, e, d);
        sm[d] = v[k];
      }
    }
  }
};

// Householder QR of the r x M panel A (stride LDA) applied to the r x W block
// X (stride LDX) -- group version of cta_householder_qr (LAPACK dlarfg
// convention, R_jj = beta).
template <int M, int W, int LDA, int LDX, int NWG>
__device__ __forceinline__ void gqr(double* A, int r, double* X, double* tau, double* rdiag, double* red, int grp,
                                    int gw, int gt) {
  constexpr int NT = NWG * 32;
#pragma unroll 1
  for (int j = 0; j < M; ++j) {
    double part = 0.0;
    for (int i = j + 1 + gt; i < r; i += NT) {
      const double v = A[i * LDA + j];
      part += v * v;
    }
    const double sig = gsum<NWG>(part, red, grp, gw);
    const double alpha = A[j * LDA + j];
    double t = 0.0, beta = alpha, scale = 0.0;
    if (sig > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + sig), alpha);
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    gsync<NWG>(grp);
    for (int i = j + 1 + gt; i < r; i += NT) A[i * LDA + j] *= scale;
    if (gt == 0) {
      tau[j] = t;
      rdiag[j] = beta;
    }
    gsync<NWG>(grp);
    const int ncols = (M - j - 1) + W;
    for (int c = gt; c < ncols; c += NT) {
      double* col;
      int ld;
      if (c < M - j - 1) {
        col = A + (j + 1 + c);
        ld = LDA;
      } else {
        col = X + (c - (M - j - 1));
        ld = LDX;
      }
      double s = col[j * ld];
      for (int i = j + 1; i < r; ++i) s += A[i * LDA + j] * col[i * ld];
      s *= t;
      col[j * ld] -= s;
      for (int i = j + 1; i < r; ++i) col[i * ld] -= s * A[i * LDA + j];
    }
    gsync<NWG>(grp);
    if (gt == 0) A[j * LDA + j] = beta;
  }
  gsync<NWG>(grp);
}

template <int N, int M, int NWG, bool SERIAL>
__device__ __forceinline__ void small_segment(const SweepArgs& a, double* sm, int grp, int gt, int64_t b, int j) {
  using S = SL<N, M>;
  constexpr int NT = NWG * 32;
  constexpr int NZ = SERIAL ? 0 : N;
  constexpr int CC = N + NZ;
  constexpr int W = CC + 1;
  constexpr int LDN = S::LDN, LDF = S::LDF, LDW = S::LDW, FW = S::FW, NN = N * N;
  const int gw = gt >> 5;
  const plq_problem_t& p = a.p;
  const int T = p.T, J = p.J;
  const int lo = p.split_times[j], hi = p.split_times[j + 1], L = hi - lo;
  double* Vxx = sm + S::V;
  double* Vzx = Vxx + N * LDN;
  double* Vzz = Vzx + N * LDN;
  double* vx1 = sm + S::VX1;
  double* vz1 = sm + S::VZ1;
  double* F = sm + S::F;
  const double* Qxx = sm + S::QXX;
  const double* Qux = sm + S::QUX;
  const double* Quu = sm + S::QUU;
  const double* qx1 = sm + S::QX1;
  const double* qu1 = sm + S::QU1;
  double* VF = sm + S::VF;
  double* P = sm + S::P;
  double* G = sm + S::G;
  double* Y = sm + S::Y;
  double* Muu = sm + S::MUU;
  double* Lm = sm + S::LM;
  double* idg = sm + S::IDG;
  double* H = sm + S::H;
  double* tau = sm + S::TAU;
  double* rdiag = sm + S::RD;
  double* red = sm + S::RED;
  int* flg = reinterpret_cast<int*>(sm + S::FLG);

  for (int idx = gt; idx < S::VZ1 + N; idx += NT) sm[idx] = 0.0;
  gsync<NWG>(grp);
  if (SERIAL) {
    for (int idx = gt; idx < NN; idx += NT) Vxx[(idx / N) * LDN + idx % N] = p.QxxT[b * NN + idx];
    for (int i = gt; i < N; i += NT) vx1[i] = p.qx1T[b * N + i];
  } else {
    for (int idx = gt; idx < N * LDW; idx += NT) {
      const int i = idx / LDW, c = idx % LDW;
      H[idx] = (c == i) ? 1.0 : ((c == N + i) ? -1.0 : 0.0);
    }
  }
  int r = SERIAL ? 0 : N;
  int status = 0;
  Prefetch<N, M, NWG> pf;
  pf.load(p, b * T + lo + L - 1, gt);
  pf.store(p, sm, gt);
  gsync<NWG>(grp);

#pragma unroll 1
  for (int s = L - 1; s >= 0; --s) {
    const int64_t st = b * T + lo + s;
    if (s > 0) pf.load(p, st - 1, gt);

    // GEMM1: [VF; Z] = [Vxx; Vzx] F; Z lands in place: Mzx -> Vzx, Mzu' -> P, mz1 -> vz1
    ggemm<N + NZ, FW, N, false, LDN, LDF, NWG>(Vxx, F, gw, [&](int i, int c, double acc) {
      if (i < N) {
        VF[i * LDF + c] = (c == N + M) ? vx1[i] + acc : acc;
      } else {
        const int zi = i - N;
        if (c < N)
          Vzx[zi * LDN + c] = acc;
        else if (c < N + M)
          P[(c - N) * LDW + N + zi] = acc;
        else
          vz1[zi] += acc;
      }
    });
    gsync<NWG>(grp);
    // GEMM2: [Mxx mx1; Mux Muu mu1] = [Fx Fu]' [VFx VFu w] + Q-blocks
    ggemm<N + M, FW, N, true, LDF, LDF, NWG>(F, VF, gw, [&](int i, int c, double acc) {
      if (i < N) {
        if (c < N)
          Vxx[i * LDN + c] = Qxx[i * N + c] + acc;
        else if (c == N + M)
          vx1[i] = qx1[i] + acc;
      } else {
        const int u = i - N;
        if (c < N)
          P[u * LDW + c] = Qux[u * N + c] + acc;
        else if (c < N + M)
          Muu[u * M + (c - N)] = Quu[u * M + (c - N)] + acc;
        else
          P[u * LDW + CC] = qu1[u] + acc;
      }
    });
    gsync<NWG>(grp);

    if (r == 0) {
      // ---- unconstrained stage: G = -Muu^{-1} P
      if (gt == 0) {
        int fail = 0;
        for (int k = 0; k < M; ++k) {
          for (int i = k; i < M; ++i) {
            double v = Muu[i * M + k];
            for (int q = 0; q < k; ++q) v -= Lm[i * M + q] * Lm[k * M + q];
            if (i == k) {
              if (!(v > 0.0)) {
                fail = 1;
                v = 1.0;
              }
              v = sqrt(v);
              Lm[k * M + k] = v;
              idg[k] = 1.0 / v;
            } else {
              Lm[i * M + k] = v * idg[k];
            }
          }
        }
        flg[0] = fail;
      }
      gsync<NWG>(grp);
      if (flg[0]) {
        status = 1 + s;
        break;
      }
      for (int c = gt; c < W; c += NT) {
        double x[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          double v = P[i * LDW + c];
#pragma unroll
          for (int k = 0; k < i; ++k) v -= Lm[i * M + k] * x[k];
          x[i] = v * idg[i];
        }
#pragma unroll
        for (int i = M - 1; i >= 0; --i) {
          double v = x[i];
#pragma unroll
          for (int k = i + 1; k < M; ++k) v -= Lm[k * M + i] * x[k];
          x[i] = v * idg[i];
        }
#pragma unroll
        for (int i = 0; i < M; ++i) G[i * LDW + c] = -x[i];
      }
      gsync<NWG>(grp);
    } else {
      // ---- constrained tail stage (r >= M since N % M == 0)
      double ph = 0.0, pu = 0.0;
      for (int idx = gt; idx < r * N; idx += NT) {
        const double v = H[(idx / N) * LDW + idx % N];
        ph += v * v;
      }
      for (int idx = gt; idx < N * M; idx += NT) {
        const double v = F[(idx / M) * LDF + N + idx % M];
        pu += v * v;
      }
      const double hx2 = gsum<NWG>(ph, red, grp, gw);
      gsync<NWG>(grp);
      const double fu2 = gsum<NWG>(pu, red, grp, gw);
      const double nu_scale = sqrt(hx2) * sqrt(fu2);
      // N = Hx F -> VF rows 0..r-1
      ggemm<N, FW, N, false, LDW, LDF, NWG>(
          H, F, gw, [&](int i, int c, double acc) { VF[i * LDF + c] = acc; }, r);
      gsync<NWG>(grp);
      for (int idx = gt; idx < r * N; idx += NT) {
        const int i = idx / N, c = idx % N;
        H[i * LDW + c] = VF[i * LDF + c];
      }
      for (int i = gt; i < r; i += NT) H[i * LDW + CC] += VF[i * LDF + N + M];
      gsync<NWG>(grp);
      gqr<M, W, LDF, LDW, NWG>(VF + N, r, H, tau, rdiag, red, grp, gw, gt);
      double rmax = 0.0, rmin = 1e308;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        rmax = fmax(rmax, fabs(rdiag[i]));
        rmin = fmin(rmin, fabs(rdiag[i]));
      }
      if (!(rmin > p.rank_tol * fmax(nu_scale, rmax))) {
        status = PLQ_STATUS_DEGENERATE;
        break;
      }
      for (int c = gt; c < W; c += NT) {
        double x[M];
#pragma unroll
        for (int i = M - 1; i >= 0; --i) {
          double v = H[i * LDW + c];
#pragma unroll
          for (int k = i + 1; k < M; ++k) v -= VF[i * LDF + N + k] * x[k];
          x[i] = v / rdiag[i];
        }
#pragma unroll
        for (int i = 0; i < M; ++i) G[i * LDW + c] = -x[i];
      }
      gsync<NWG>(grp);
      for (int blk = 0; blk < r - M; blk += M) {
        const int rows = min(M, r - M - blk);
        for (int idx = gt; idx < rows * W; idx += NT) {
          const int i = blk + idx / W, c = idx % W;
          H[i * LDW + c] = H[(i + M) * LDW + c];
        }
        gsync<NWG>(grp);
      }
      r -= M;
    }

    // ---- policy outputs
    for (int idx = gt; idx < M * N; idx += NT) {
      const int u = idx / N, c = idx % N;
      a.Kx[st * (M * N) + idx] = G[u * LDW + c];
      a.Kz[st * (M * N) + idx] = SERIAL ? 0.0 : G[u * LDW + N + c];
    }
    for (int u = gt; u < M; u += NT) a.k1[st * M + u] = G[u * LDW + CC];

    // ---- value update: Y = P + Muu G ; V += P'G + G'Y
    ggemm<M, W, M, false, M, LDW, NWG>(Muu, G, gw,
                                       [&](int i, int c, double acc) { Y[i * LDW + c] = P[i * LDW + c] + acc; });
    gsync<NWG>(grp);
    ggemm<N + NZ, W, 2 * M, true, LDW, LDW, NWG>(P, G, gw, [&](int i, int c, double acc) {
      if (i < N) {
        if (c < N)
          Vxx[i * LDN + c] += acc;
        else if (c == CC)
          vx1[i] += acc;
      } else {
        const int zi = i - N;
        if (c < N)
          Vzx[zi * LDN + c] += acc;
        else if (c < CC)
          Vzz[zi * LDN + (c - N)] += acc;
        else
          vz1[zi] += acc;
      }
    });
    gsync<NWG>(grp);
    for (int idx = gt; idx < NN; idx += NT) {
      const int i = idx / N, c = idx % N;
      if (i < c) {
        const double v = 0.5 * (Vxx[i * LDN + c] + Vxx[c * LDN + i]);
        Vxx[i * LDN + c] = v;
        Vxx[c * LDN + i] = v;
        if (!SERIAL) {
          const double w = 0.5 * (Vzz[i * LDN + c] + Vzz[c * LDN + i]);
          Vzz[i * LDN + c] = w;
          Vzz[c * LDN + i] = w;
        }
      }
    }
    if (s > 0) pf.store(p, sm, gt);
    gsync<NWG>(grp);
  }

  const int vsz = 3 * NN + 2 * N;
  double* dst = a.vf0 + (b * J + j) * (int64_t)vsz;
  for (int idx = gt; idx < 3 * NN; idx += NT) {
    const int blk = idx / NN, e = idx % NN;
    dst[idx] = sm[S::V + blk * N * LDN + (e / N) * LDN + e % N];
  }
  for (int i = gt; i < 2 * N; i += NT) dst[3 * NN + i] = sm[S::VX1 + i];
  if (gt == 0) {
    if (status == 0 && !SERIAL && r > 0) status = PLQ_STATUS_DEGENERATE;
    a.status[b * J + j] = status;
  }
  gsync<NWG>(grp);
}

template <int N, int M, int NWG, int GROUPS>
__global__ void __launch_bounds__(NWG * 32 * GROUPS) sweep_small_kernel(SweepArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int grp = threadIdx.x / (NWG * 32);
  const int gt = threadIdx.x % (NWG * 32);
  double* sm = smem + grp * SL<N, M>::TOTAL;
  const int nloc = a.seg_end - a.seg_begin;
  const int64_t total = a.p.B * nloc;
  for (int64_t task = (int64_t)blockIdx.x * GROUPS + grp; task < total; task += (int64_t)gridDim.x * GROUPS) {
    const int64_t b = task / nloc;
    const int j = a.seg_begin + (int)(task % nloc);
    if (j == a.p.J - 1)
      small_segment<N, M, NWG, true>(a, sm, grp, gt, b, j);
    else
      small_segment<N, M, NWG, false>(a, sm, grp, gt, b, j);
  }
}

template <int N, int M, int NWG, int GROUPS>
int launch_small(const SweepArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(double) * SL<N, M>::TOTAL * GROUPS;
  auto kern = sweep_small_kernel<N, M, NWG, GROUPS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NWG * 32 * GROUPS, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tasks = a.p.B * (int64_t)(a.seg_end - a.seg_begin);
  const int64_t blocks_needed = (tasks + GROUPS - 1) / GROUPS;
  const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(blocks_needed < cap ? blocks_needed : cap);
  kern<<<grid, NWG * 32 * GROUPS, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace

bool sweep_small_supported(int n, int m) { return (n == 12 && m == 4) || (n == 32 && m == 8); }

int launch_sweep_small(const SweepArgs& a, cudaStream_t s) {
  if (a.p.n == 12 && a.p.m == 4) return launch_small<12, 4, 1, 1>(a, s);
  if (a.p.n == 32 && a.p.m == 8) return launch_small<32, 8, 4, 1>(a, s);
  return -1;
}

}  // namespace plq
