// K1 specialized: segment sweeps with compile-time n, m (BASELINE configs
// 0-2 and 4: n=12/m=4, n=32/m=8, n=64/m=32).  n = 64 ("BIG") keeps the GEMM
// operands on chip and the rest in L2 scratch, uses the blocked
// factorizations of plq_blocked.cuh and tile-selective GEMMs.
//
// Same recurrences as the generic sweep (plq_sweep.cu; endpoint.py:168-301,
// serial.py:37-79), restructured for latency:
//   * one group of NWG warps per segment, group barriers only;
//   * each stage's inputs arrive by bulk asynchronous copy (TMA 1-D,
//     cp.async.bulk) into a shared staging buffer; the copy for stage s-1 is
//     issued as soon as stage s has consumed its inputs, so it overlaps the
//     gain / value-update half of the stage;
//   * GEMM operands are read straight from the staged fields ([Fx|Fu|f1] by a
//     loader functor) -- no re-layout pass; other buffers use strides = 4
//     (mod 8) doubles so the DMMA fragment loads are bank-conflict free;
//   * GEMM epilogues write in place: GEMM1 puts Mzx straight into Vzx (band
//     by band -- a band only reads its own rows) and Mzu' into P, GEMM2 puts
//     Mxx/mx1 into Vxx/vx1, and the value update accumulates into V;
//   * the m x m Cholesky of Muu is computed redundantly in every lane's
//     registers (m <= 8), so the gain solve needs no barrier.
#include "plq_blocked.cuh"
#include "plq_gemm.cuh"
#include "plq_internal.h"
#include "plq_small.cuh"
#include "plq_tma.cuh"

namespace plq {

// Optional per-phase cycle accounting (build with -DPLQ_PHASE_PROFILE; a
// measurement build only): group 0 thread 0 of every CTA adds clock64()
// deltas per stage phase into g_phase_cycles[blockIdx.x][phase].
#ifdef PLQ_PHASE_PROFILE
__device__ unsigned long long g_phase_cycles[1024][16];
#define PLQ_PHASE(k)                                                               \
  do {                                                                             \
    if (gt == 0) {                                                                 \
      const long long t_ = clock64();                                              \
      atomicAdd(&g_phase_cycles[blockIdx.x & 1023][k], (unsigned long long)(t_ - t_last)); \
      t_last = t_;                                                                 \
    }                                                                              \
  } while (0)
#else
#define PLQ_PHASE(k) \
  do {               \
  } while (0)
#endif

namespace {

template <int N, int M>
struct SL {
  // BIG (n >= 64): only the GEMM operands stay in shared memory ([Vxx;Vzx],
  // staged [Fx|Fu|f1], VF / G, P, Muu); Vzz, the constraint rows H, Y and the
  // tail temporaries live in a per-CTA slice of (L2-resident) global scratch,
  // and the Q blocks are read from global memory in the GEMM2 epilogue.
  static constexpr bool BIG = N >= 64;
  // QREG (n <= 16, single-warp groups): the Q blocks are not staged; each lane
  // prefetches the Q values of its own GEMM2 epilogue fragments into registers
  static constexpr bool QREG = N <= 16;
  static constexpr bool QSTAGED = !BIG && !QREG;
  static constexpr int NN = N * N, NM = N * M, MM = M * M;
  static constexpr int LDN = pad_ld(N);
  static constexpr int FW = N + M + 1;
  static constexpr int LDF = pad_ld(FW);
  static constexpr int WE = 2 * N + 1;
  static constexpr int LDW = pad_ld(WE);
  static constexpr int LDM = pad_ld(M);
  // Fx rows are staged row by row with a padded stride when N is not already
  // conflict-free (N % 8 != 4)
  static constexpr bool FX_ROWS = (N % 8) != 4;
  static constexpr int LFX = FX_ROWS ? pad_ld(N) : N;
  static constexpr bool FU_ROWS = (M % 8) != 4 && M > 4;
  static constexpr int LFU = FU_ROWS ? pad_ld(M) : M;
  static constexpr int V = 0;                    // Vxx, Vzx (, Vzz): (BIG ? 2 : 3) x (N x LDN)
  static constexpr int VX1 = V + (BIG ? 2 : 3) * N * LDN;
  static constexpr int VZ1 = VX1 + N;
  // staged stage inputs (16-byte aligned fields)
  static constexpr int SFX = (VZ1 + N + 1) & ~1;        // N x LFX
  static constexpr int SFU = SFX + N * LFX;             // N x LFU
  static constexpr int SF1 = SFU + N * LFU;             // N
  static constexpr int SQXX = SF1 + N;                  // N x N  (not BIG)
  static constexpr int SQUX = SQXX + (QSTAGED ? NN : 0);    // M x N
  static constexpr int SQUU = SQUX + (QSTAGED ? NM : 0);    // M x M
  static constexpr int SQX1 = SQUU + (QSTAGED ? MM : 0);    // N
  static constexpr int SQU1 = SQX1 + (QSTAGED ? N : 0);     // M
  static constexpr int VF = (SQU1 + (QSTAGED ? M : 0) + 1) & ~1;   // N x LDF (also N = Hx F)
  static constexpr int P = VF + N * LDF;                // P (then G, Y when not BIG): M x LDW each
  static constexpr int G = BIG ? VF : P + M * LDW;      // BIG: G overlays VF (dead after GEMM2)
  static constexpr int Y = BIG ? -1 : G + M * LDW;
  static constexpr int MUU = (BIG ? P + M * LDW : Y + M * LDW);   // M x LDM
  static constexpr int H = MUU + M * LDM;               // N x LDW constraint rows (not BIG)
  static constexpr int TAU = H + (BIG ? 0 : N * LDW);   // M x M (tau, or the WY factor T)
  static constexpr int RD = TAU + M * M;                // M
  static constexpr int RED = RD + M;                    // 8
  static constexpr int DUM = RED + 8;                   // 32 per-lane dummy slots (branch-free epilogues)
  static constexpr int BAR = (DUM + 32 + 1) & ~1;       // mbarrier (8 bytes)
  static constexpr int FLAG = BAR + 2;                  // int flag of the blocked Cholesky (BIG)
  static constexpr int TOTAL = FLAG + 2;
  // global scratch per CTA (BIG): Vzz (N x LDN), H (N x LDW), Y (M x LDW)
  static constexpr int GVZZ = 0, GH = GVZZ + N * LDN, GY = GH + N * LDW;
  static constexpr int GTOTAL = BIG ? GY + M * LDW : 0;
  static constexpr uint32_t STAGE_BYTES = QSTAGED ? 8u * (2 * NN + 2 * NM + MM + 2 * N + M) : 8u * (NN + NM + N);
  static_assert(SFX % 2 == 0 && SFU % 2 == 0 && SF1 % 2 == 0 && SQXX % 2 == 0 && SQUX % 2 == 0 &&
                    SQUU % 2 == 0 && SQX1 % 2 == 0 && SQU1 % 2 == 0 && (N * 8) % 16 == 0 && (M * 8) % 16 == 0,
                "bulk copies need 16-byte alignment");
};

// Stage `st`'s inputs into the staging fields, issued by EVERY thread of the
// group (all must call).  Contiguous fields go by one bulk copy each (TMA
// 1-D, complete_tx on the stage mbarrier); the row-padded Fx / Fu layouts
// (n = 32, 64: conflict-free DMMA fragment strides) go by 16-byte cp.async
// spread over the group, each thread then arriving on the same mbarrier when
// its copies land (cp.async.mbarrier.arrive.noinc; the barrier counts 1 + NT
// arrivals).  One bulk copy per row instead -- ~130 UBLKCP per n = 64 stage,
// ~70 at n = 32 -- was issue-bound (measured: ~4k cycles per n = 32 stage).
template <int N, int M>
__host__ __device__ constexpr uint32_t stage_bulk_bytes() {
  using S = SL<N, M>;
  return S::STAGE_BYTES - (S::FX_ROWS ? 8u * N * N : 0u) - (S::FU_ROWS ? 8u * N * M : 0u);
}

template <int N, int M, int NT>
__device__ __forceinline__ void stage_issue_group(const plq_problem_t& p, int64_t st, double* sm, uint64_t* bar,
                                                  int gt) {
  using S = SL<N, M>;
  constexpr int NN = N * N, NM = N * M, MM = M * M;
  if (gt < 8) fence_proxy_async();   // the bulk-copy issuers: generic reads before async writes
  if (gt == 0) mbar_arrive_tx(bar, stage_bulk_bytes<N, M>());
  if constexpr (S::FX_ROWS) {
    constexpr int CR = N / 2;   // 16-byte chunks per row
    const double* src = p.Fx + st * NN;
#pragma unroll 1
    for (int c = gt; c < N * CR; c += NT) cp_async16(sm + S::SFX + (c / CR) * S::LFX + 2 * (c % CR), src + 2 * c);
  } else if (gt == 0) {
    bulk_g2s(sm + S::SFX, p.Fx + st * NN, 8u * NN, bar);
  }
  if constexpr (S::FU_ROWS) {
    constexpr int CR = M / 2;
    const double* src = p.Fu + st * NM;
#pragma unroll 1
    for (int c = gt; c < N * CR; c += NT) cp_async16(sm + S::SFU + (c / CR) * S::LFU + 2 * (c % CR), src + 2 * c);
  } else if (gt == (NT > 1 ? 1 : 0)) {
    bulk_g2s(sm + S::SFU, p.Fu + st * NM, 8u * NM, bar);
  }
  const int lane = gt & 31;
  if (gt < 32) {
    if (lane == 2 % NT) bulk_g2s(sm + S::SF1, p.f1 + st * N, 8u * N, bar);
    if constexpr (S::BIG) {
      // the Q blocks are not staged (GEMM2 loads them as epilogue addends):
      // pull them into L2 now, a stage ahead, so those loads hit L2 not HBM
      if (lane == 3) bulk_prefetch_l2(p.Qxx + st * NN, 8u * NN);
      if (lane == 4) bulk_prefetch_l2(p.Qux + st * NM, 8u * NM);
      if (lane == 5) bulk_prefetch_l2(p.Quu + st * MM, 8u * MM);
      if (lane == 6) bulk_prefetch_l2(p.qx1 + st * N, 8u * N);
      if (lane == 7) bulk_prefetch_l2(p.qu1 + st * M, 8u * M);
    }
    if constexpr (S::QSTAGED) {
      if (lane == 3) bulk_g2s(sm + S::SQXX, p.Qxx + st * NN, 8u * NN, bar);
      if (lane == 4) bulk_g2s(sm + S::SQUX, p.Qux + st * NM, 8u * NM, bar);
      if (lane == 5) bulk_g2s(sm + S::SQUU, p.Quu + st * MM, 8u * MM, bar);
      if (lane == 6) bulk_g2s(sm + S::SQX1, p.qx1 + st * N, 8u * N, bar);
      if (lane == 7) bulk_g2s(sm + S::SQU1, p.qu1 + st * M, 8u * M, bar);
    }
  }
  cp_async_arrive_noinc(bar);
}

// F(k, j) = [Fx | Fu | f1](k, j) from the staged fields
template <int N, int M>
__device__ __forceinline__ double fload(const double* sm, int k, int j) {
  using S = SL<N, M>;
  // one address select, one load
  const int off = (j < N) ? S::SFX + k * S::LFX + j : ((j < N + M) ? S::SFU + k * S::LFU + (j - N) : S::SF1 + k);
  return sm[off];
}

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

// Householder QR of the r x M panel (r <= 32, M <= 8) held one row per lane
// in registers (LAPACK dlarfg convention, as cta_householder_qr), then
// Q' X for the r x W block X via the compact WY form Q' = I - V T' V'
// (dlarft): y = V'x, z = T'y, x -= V z per column -- independent
// dot products instead of M sequential reflector sweeps.  R (upper) and V
// (strictly lower, unit diagonal implicit) are written back LAPACK-style to
// A; rdiag gets diag(R).
template <int M, int W, int LDA, int LDX, int RMAX>
__device__ __forceinline__ void warp_qr_wy(double* A, int r, double* X, double* Tm, double* rdiag, double* VTs,
                                           double* Ys) {
  const int lane = threadIdx.x & 31;
  const bool row = lane < r;
  // rows live in lanes < r <= RMAX: for RMAX <= 16 a half-warp butterfly is
  // the full sum for lanes 0-15 (lanes 16-31 hold zeros, never use it)
  auto warp_sum = [&](double x) {
    if constexpr (RMAX <= 16) {
#pragma unroll
      for (int o = 8; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      return x;
    } else {
      return plq::warp_sum(x);
    }
  };
  double a[M], v[M], tau[M];
#pragma unroll
  for (int k = 0; k < M; ++k) a[k] = row ? A[lane * LDA + k] : 0.0;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const double x = (lane > j && row) ? a[j] : 0.0;
    const double sig = warp_sum(x * x);
    const double alpha = __shfl_sync(0xffffffffu, a[j], j);
    double t = 0.0, beta = alpha, scale = 0.0;
    if (sig > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + sig), alpha);
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    const double vj = (lane == j) ? 1.0 : ((lane > j && row) ? a[j] * scale : 0.0);
    v[j] = vj;
    tau[j] = t;
#pragma unroll
    for (int k = j + 1; k < M; ++k) {
      const double sk = warp_sum(vj * a[k]);
      if (lane >= j) a[k] -= t * sk * vj;
    }
    if (lane == j) a[j] = beta;
    if (lane == 0) rdiag[j] = beta;
  }
  // write R (upper) and V (strictly lower) back in place
  if (row) {
#pragma unroll
    for (int k = 0; k < M; ++k) A[lane * LDA + k] = (k >= lane) ? a[k] : v[k];
  }
  // T (upper triangular, M x M): T_jj = tau_j, T[0:j, j] = -tau_j T[0:j,0:j] V[:,0:j]' v_j
  double vtv[M][M];
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = i + 1; j < M; ++j) vtv[i][j] = warp_sum(v[i] * v[j]);
  if (lane == 0) {
    double T[M][M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
#pragma unroll
      for (int i = 0; i < M; ++i) T[i][j] = 0.0;
      T[j][j] = tau[j];
#pragma unroll
      for (int i = 0; i < j; ++i) {
        double t = 0.0;
#pragma unroll
        for (int k = i; k < j; ++k) t += T[i][k] * vtv[k][j];
        T[i][j] = -tau[j] * t;
      }
    }
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < M; ++j) Tm[i * M + j] = T[i][j];
  }
  __syncwarp();
  // X <- X - (V T') (V' X) on the FP64 tensor pipe: Y = V'X (M x W, K = r),
  // VT = V T' (r x M, each row-lane from its own v), X -= VT Y (r x W, K = M).
  // V' rows are read back from A (unit diagonal, zeros above); rows >= r are 0.
  ggemm_f<M, W, RMAX, 1>(
      [&](int i, int k) { return (k == i) ? 1.0 : ((k > i && k < r) ? A[k * LDA + i] : 0.0); },
      [&](int k, int c) { return k < r ? X[k * LDX + c] : 0.0; }, 0,
      [&](int i, int c, double acc) { Ys[i * LDX + c] = acc; });
  if (row) {
#pragma unroll
    for (int j = 0; j < M; ++j) {
      double t = 0.0;
#pragma unroll
      for (int l = j; l < M; ++l) t += v[l] * Tm[j * M + l];   // (V T')_{lane, j}, T upper
      VTs[lane * LDA + j] = t;
    }
  }
  __syncwarp();
  ggemm_f<RMAX, W, M, 1>([&](int i, int k) { return VTs[i * LDA + k]; }, [&](int k, int c) { return Ys[k * LDX + c]; },
                         0, [&](int i, int c, double acc) { X[i * LDX + c] -= acc; }, r);
  __syncwarp();
}

template <int N, int M, int NWG, bool SERIAL>
__device__ __forceinline__ void small_segment(const SweepArgs& a, double* sm, int grp, int gt, int64_t b, int j,
                                              uint32_t& phase, const unsigned short* pairs) {
  constexpr int NP = N * (N - 1) / 2;
  using S = SL<N, M>;
  constexpr int NT = NWG * 32;
  constexpr int NZ = SERIAL ? 0 : N;
  constexpr int CC = N + NZ;
  constexpr int W = CC + 1;
  constexpr int LDN = S::LDN, LDF = S::LDF, LDW = S::LDW, FW = S::FW, NN = N * N;
  const int gw = gt >> 5;
  const int lane = threadIdx.x & 31;
  const plq_problem_t& p = a.p;
  const int T = p.T, J = p.J;
  const int lo = p.split_times[j], hi = p.split_times[j + 1], L = hi - lo;
  constexpr int LDM = S::LDM;
  // tile-selective GEMM2 / value update (symmetric blocks computed once)
  constexpr bool SEL = S::BIG && N == 64 && M == 32 && NWG == 8;
  constexpr int XB = N / 8;
  double* gs = a.gscratch + (int64_t)blockIdx.x * S::GTOTAL;   // BIG: per-CTA L2 scratch
  double* Vxx = sm + S::V;
  double* Vzx = Vxx + N * LDN;
  double* Vzz = S::BIG ? gs + S::GVZZ : Vzx + N * LDN;
  double* vx1 = sm + S::VX1;
  double* vz1 = sm + S::VZ1;
  double* VF = sm + S::VF;
  double* P = sm + S::P;
  double* G = sm + S::G;
  double* Y = S::BIG ? gs + S::GY : sm + S::Y;
  double* Muu = sm + S::MUU;
  double* H = S::BIG ? gs + S::GH : sm + S::H;
  double* NTb = VF;   // tail-stage N = Hx F (G, which overlays VF when BIG, is written after R is copied out)
  double* tau = sm + S::TAU;
  double* rdiag = sm + S::RD;
  double* red = sm + S::RED;
  // per-lane sink for skipped epilogue elements (QREG: unused VF padding columns)
  double* dum = S::QREG ? sm + S::VF + (lane % N) * S::LDF + S::FW + lane / N : sm + S::DUM + lane;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::BAR);

  stage_issue_group<N, M, NT>(p, b * T + lo + L - 1, sm, bar, gt);
  for (int idx = gt; idx < S::VZ1 + N; idx += NT) sm[idx] = 0.0;
  if constexpr (S::BIG)
    for (int idx = gt; idx < N * LDN; idx += NT) Vzz[idx] = 0.0;
  gsync<NWG>(grp);
  if (SERIAL && a.smooth_vf0) {
    // smoothing pass: TerminalCost(Vxx, vx1 + Vzx' z) of segment j+1 (parallel.py:598-606)
    const double* v = a.smooth_vf0 + (b * J + j + 1) * (int64_t)(3 * NN + 2 * N);
    const double* z = a.smooth_links + (b * (J - 1) + j + 1) * (int64_t)N;
    for (int idx = gt; idx < NN; idx += NT) {
      const int i = idx / N, c = idx % N;
      Vxx[i * LDN + c] = 0.5 * (v[i * N + c] + v[c * N + i]);
    }
    for (int i = gt; i < N; i += NT) {
      double t = 0.0;
      if (j + 1 < J - 1)
        for (int k = 0; k < N; ++k) t += v[NN + k * N + i] * z[k];
      vx1[i] = v[3 * NN + i] + t;
    }
  } else if (SERIAL) {
    for (int idx = gt; idx < NN; idx += NT) Vxx[(idx / N) * LDN + idx % N] = p.QxxT[b * NN + idx];
    for (int i = gt; i < N; i += NT) vx1[i] = p.qx1T[b * N + i];
  } else {
    for (int idx = gt; idx < N * LDW; idx += NT) {
      const int i = idx / LDW, c = idx % LDW;
      H[idx] = (c == i) ? 1.0 : ((c == N + i) ? -1.0 : 0.0);
    }
    if (a.endpoint_terminal && j == J - 1) {   // terminal cost + terminal rows (endpoint.py:178-191)
      for (int idx = gt; idx < NN; idx += NT) {
        const int i = idx / N, c = idx % N;
        Vxx[i * LDN + c] = 0.5 * (p.QxxT[b * NN + i * N + c] + p.QxxT[b * NN + c * N + i]);
      }
      for (int i = gt; i < N; i += NT) vx1[i] = p.qx1T[b * N + i];
    }
  }
  int r = SERIAL ? 0 : N;
  int status = 0;
  // QREG: Q values of this lane's GEMM2 epilogue slots (+ its qx1 / qu1 entry)
  constexpr int QS = S::QREG ? ((N + M + 7) / 8) * ((N + M + 7) / 8) * 2 : 1;
  double qv[QS], qw = 0.0;
  auto q_prefetch = [&](int64_t stq) {
    if constexpr (S::QREG) {
      const int g = lane >> 2, q4 = lane & 3;
      constexpr int TN2 = (N + M + 7) / 8;
#pragma unroll
      for (int sl = 0; sl < QS; ++sl) {
        const int tm = sl / (2 * TN2), tn = (sl / 2) % TN2, e = sl & 1;
        const int i = tm * 8 + g, c = tn * 8 + 2 * q4 + e;
        double v = 0.0;
        if (i < N + M && c < N + M) {
          const int u = i - N;
          v = (i < N) ? (c < N ? __ldg(p.Qxx + stq * NN + i * N + c) : 0.0)
                      : (c < N ? __ldg(p.Qux + stq * (N * M) + u * N + c) : __ldg(p.Quu + stq * (M * M) + u * M + (c - N)));
        }
        qv[sl] = v;
      }
      qw = gt < N ? __ldg(p.qx1 + stq * N + gt) : (gt < N + M ? __ldg(p.qu1 + stq * M + gt - N) : 0.0);
    }
  };
  q_prefetch(b * T + lo + L - 1);
  gsync<NWG>(grp);

#ifdef PLQ_PHASE_PROFILE
  long long t_last = clock64();
#endif
#pragma unroll 1
  for (int s = L - 1; s >= 0; --s) {
    const int64_t st = b * T + lo + s;
    const double* Qxx = S::QSTAGED ? sm + S::SQXX : p.Qxx + st * NN;
    const double* Qux = S::QSTAGED ? sm + S::SQUX : p.Qux + st * (N * M);
    const double* Quu = S::QSTAGED ? sm + S::SQUU : p.Quu + st * (M * M);
    const double* qx1 = S::QSTAGED ? sm + S::SQX1 : p.qx1 + st * N;
    const double* qu1 = S::QSTAGED ? sm + S::SQU1 : p.qu1 + st * M;
    PLQ_PHASE(8);   // end of the previous stage / segment prologue
    mbar_wait(bar, phase);
    phase ^= 1u;
    PLQ_PHASE(0);   // stage-input copy wait

    // GEMM1: [VF; Z] = [Vxx; Vzx] [Fx | Fu]; Z lands in place: Mzx -> Vzx, Mzu' -> P.
    // The f1 column (w = vx1 + Vxx f1, mz1 = vz1 + Vzx f1) is a lane-parallel
    // dot product instead of a mostly empty 8-wide DMMA tile; it reads Vzx
    // before the in-place epilogue overwrites it.
    double wcol = 0.0;
    const bool wrow = gt < N + NZ;
    if (wrow) {
      const double* vr = Vxx + gt * LDN;
      double w2 = 0.0;
      if constexpr (N % 16 == 0) {
        // The row stride (= 4 mod 8 doubles, chosen for the DMMA fragment loads)
        // puts lanes l and l + 4 of a plain vr[k] load on the same banks (8-way
        // conflict).  16-byte loads starting at column pair (c - l) spread every
        // quarter-warp over all eight 16-byte bank groups.
        const double2* v2 = reinterpret_cast<const double2*>(vr);
        const double2* f2 = reinterpret_cast<const double2*>(sm + S::SF1);
#pragma unroll 8
        for (int c = 0; c < N / 2; ++c) {
          const int k2 = (c - gt) & (N / 2 - 1);
          const double2 av = v2[k2], fv = f2[k2];
          wcol += av.x * fv.x;
          w2 += av.y * fv.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < N; k += 2) {
          wcol += vr[k] * sm[S::SF1 + k];
          w2 += vr[k + 1] * sm[S::SF1 + k + 1];
        }
      }
      wcol += w2;
    }
    gsync<NWG>(grp);
    PLQ_PHASE(1);   // f1 column dot products
    ggemm_f<N + NZ, N + M, N, NWG>(
        [&](int i, int k) { return Vxx[i * LDN + k]; }, [&](int k, int c) { return fload<N, M>(sm, k, c); }, gw,
        [&](int i, int c, double acc) {
          const int zi = i - N;
          double* d = (i < N) ? VF + i * LDF + c : ((c < N) ? Vzx + zi * LDN + c : P + (c - N) * LDW + N + zi);
          *d = acc;
        });
    PLQ_PHASE(14);   // GEMM1 k-loops (warp 0's bands)
    if (wrow) {
      if (gt < N)
        VF[gt * LDF + N + M] = vx1[gt] + wcol;
      else
        vz1[gt - N] += wcol;
    }
    gsync<NWG>(grp);
    PLQ_PHASE(2);   // GEMM1
    // GEMM2: [Mxx ; Mux Muu] = [Fx Fu]' [VFx VFu] + Q-blocks; the w column
    // (mx1 = qx1 + Fx' w, mu1 = qu1 + Fu' w) lane-parallel
    if constexpr (S::QREG) {
      wgemm_slots<N + M, N + M, N>(
          [&](int i, int k) { return fload<N, M>(sm, k, i); }, [&](int k, int c) { return VF[k * LDF + c]; },
          [&](int i, int c, double acc, int slot) {
            const int u = i - N;
            const bool xr = i < N, xc = c < N;
            double* d = xr ? (xc ? Vxx + i * LDN + c : dum) : (xc ? P + u * LDW + c : Muu + u * LDM + (c - N));
            *d = qv[slot] + acc;
          });
    } else if constexpr (SEL) {
      // x bands: the lower triangle of Mxx only (the value update mirrors
      // V), no Mxu block; u bands: Mux | Muu in full.  Warps 0-3 take a u
      // band (12 tiles), warps 4-7 a pair of x bands (9 tiles).  The Q-block
      // addends are loaded from global memory before each band's k-loop.
      auto fa = [&](int i, int k) { return fload<N, M>(sm, k, i); };
      auto fb = [&](int k, int c) { return VF[k * LDF + c]; };
      auto on2 = [](int tm, int tn) { return tm >= XB || tn <= tm; };
      auto qpre = [&](int i, int c) {
        const int u = i - N;
        return i < N ? __ldg(Qxx + i * N + c) : (c < N ? __ldg(Qux + u * N + c) : __ldg(Quu + u * M + (c - N)));
      };
      auto mepi = [&](int i, int c, double v, bool) {
        const int u = i - N;
        if (i < N) {
          if (c <= i) Vxx[i * LDN + c] = v;
        } else if (c < N) {
          P[u * LDW + c] = v;
        } else {
          Muu[u * LDM + (c - N)] = v;
        }
      };
      // warps 0-3: one u band; warps 4-7: an x-band pair in one k-loop
      // (bands fixed per warp at compile time: no runtime tile predicates)
      auto g2 = [&](auto w) {
        constexpr int WI = decltype(w)::value;
        if constexpr (WI < 4)
          ggemm_sel2<N + M, N + M, N, (N + M) / 8, 0, true, 0, XB + WI, -1>(fa, fb, on2, qpre, mepi);
        else
          ggemm_sel2<N + M, N + M, N, XB, XB, true, 0, WI - 4, XB + 3 - WI>(fa, fb, on2, qpre, mepi);
      };
      warp_dispatch8(gw, g2);
      PLQ_PHASE(12);   // GEMM2 k-loops (warp 0's band)
    } else {
      ggemm_f<N + M, N + M, N, NWG>(
          [&](int i, int k) { return fload<N, M>(sm, k, i); }, [&](int k, int c) { return VF[k * LDF + c]; }, gw,
          [&](int i, int c, double acc) {
            const int u = i - N;
            const bool xr = i < N, xc = c < N;
            const double* q = xr ? Qxx + i * N + (xc ? c : 0) : (xc ? Qux + u * N + c : Quu + u * M + (c - N));
            double* d = xr ? (xc ? Vxx + i * LDN + c : dum) : (xc ? P + u * LDW + c : Muu + u * LDM + (c - N));
            *d = *q + acc;
          });
    }
    if (gt < N + M) {
      double t = 0.0, t2 = 0.0;
#pragma unroll
      for (int k = 0; k < N; k += 2) {
        t += fload<N, M>(sm, k, gt) * VF[k * LDF + N + M];
        t2 += fload<N, M>(sm, k + 1, gt) * VF[(k + 1) * LDF + N + M];
      }
      t += t2;
      const double qg = S::QREG ? qw : (gt < N ? qx1[gt] : qu1[gt - N]);
      if (gt < N)
        vx1[gt] = qg + t;
      else
        P[(gt - N) * LDW + CC] = qg + t;
    }
    if (s > 0) q_prefetch(st - 1);   // next stage's Q values, consumed one stage later

    gsync<NWG>(grp);
    PLQ_PHASE(3);   // GEMM2

    const bool constrained = (r != 0);
    bool chol = !constrained;
    if (constrained) {
      // ---- constrained tail stage (r >= M since N % M == 0)
      double ph = 0.0, pu = 0.0;
      for (int idx = gt; idx < r * N; idx += NT) {
        const double v = H[(idx / N) * LDW + idx % N];
        ph += v * v;
      }
      for (int idx = gt; idx < N * M; idx += NT) {
        const double v = sm[S::SFU + (idx / M) * S::LFU + idx % M];
        pu += v * v;
      }
      const double hx2 = gsum<NWG>(ph, red, grp, gw);
      gsync<NWG>(grp);
      const double fu2 = gsum<NWG>(pu, red, grp, gw);
      const double nu_scale = sqrt(hx2) * sqrt(fu2);
      // N = Hx F, stacked in place: [Nx | Hz | Hx f1 + h1] into H, Nu into
      // NTb (every band's loads precede its stores; bands own their rows)
      ggemm_f<N, FW, N, NWG>(
          [&](int i, int k) { return H[i * LDW + k]; }, [&](int k, int c) { return fload<N, M>(sm, k, c); }, gw,
          [&](int i, int c, double acc) {
            if (c < N)
              H[i * LDW + c] = acc;
            else if (c < N + M)
              NTb[i * LDF + c] = acc;
            else
              H[i * LDW + CC] += acc;
          },
          r);
      gsync<NWG>(grp);
      PLQ_PHASE(10);   // tail: norms + N = Hx F
      if (s > 0) stage_issue_group<N, M, NT>(p, st - 1, sm, bar, gt);   // F consumed
      if constexpr (NWG == 1) {
        // tau slot holds T (M*M); NTb columns 0..M-1 (free: Nx went to H) take V T',
        // the Y slot (dead until the value update) takes V'X
        warp_qr_wy<M, W, LDF, LDW, N>(NTb + N, r, H, tau, rdiag, NTb, Y);
      } else if constexpr (S::BIG) {
        // blocked compact-WY QR: the TAU slot (M*M >= 8N + 8*64 doubles) holds
        // V T' and the per-warp tiles
        static_assert(M * M >= N * 8 + NWG * 64, "TAU slot too small for the blocked QR");
        auto sy = [&] { gsync<NWG>(grp); };
        gqr8<NWG, decltype(sy), (N + 31) / 32>(NTb + N, r, M, LDF, H, W, LDW, rdiag, tau, tau + N * 8, gt, sy);
      } else {
        // n = 32 (M = 8, one panel, H on chip): the column-wise group QR
        // (measured faster here than gqr8: 2.46 vs 2.51 ms cfg2 sweep)
        gqr<M, W, LDF, LDW, NWG>(NTb + N, r, H, tau, rdiag, red, grp, gw, gt);
      }
      PLQ_PHASE(11);   // tail: QR of Nu applied to the rows
      // rank certificates (plq_rank.cuh): p = 0 for sure when ||R||_F <= thr,
      // p = M for sure when 1 / ||R^{-1}||_F = 1 / ||Kz||_F > thr; anything
      // else is re-solved by the rank-revealing repair pass (SVD decision,
      // the reference's endpoint.py:226-231)
      const double* Rm = NTb + N;   // R (upper) with stride LDF
      double rmax = 0.0, pf = 0.0;
#pragma unroll
      for (int i = 0; i < M; ++i) rmax = fmax(rmax, fabs(rdiag[i]));
      for (int idx = gt; idx < M * M; idx += NT) {
        const int i = idx / M, c = idx % M;
        const double v = c > i ? Rm[i * LDF + c] : (c == i ? rdiag[i] : 0.0);
        pf += v * v;
      }
      const double thr = p.rank_tol * fmax(nu_scale, rmax);
      double rf2 = 0.0;
      if constexpr (S::BIG) {
        // the blocked back substitution below overwrites H's first M rows,
        // which a p = 0 stage keeps: decide p = 0 first
        rf2 = gsum<NWG>(pf, red, grp, gw);
        gsync<NWG>(grp);
      }
      if (S::BIG && sqrt(rf2) <= thr) {
        // p = 0 (Nu numerically zero): identity reflectors, all r rows stay,
        // gains by the null-space solve with Zw = I (endpoint.py:239-250)
        chol = true;
      } else {
        int ldr = LDF;
        double pz = 0.0;   // ||Kz||_F^2 partial (the z columns of G)
        if constexpr (S::BIG) {
          // G = -R^{-1} (Q1' stack): blocked back substitution in place on
          // H's first M rows (R stays in NTb, which G overlays), then G = -H
          auto sy = [&] { gsync<NWG>(grp); };
          gtri_inv_upper8<NWG>(Rm, M, ldr, rdiag, tau, gt, sy);
          gtrsm8<2, NWG>(Rm, M, ldr, tau, H, W, LDW, tau + 256, gt, sy);
          for (int idx = gt; idx < M * W; idx += NT) {
            const int c = idx % W;
            const double g = -H[(idx / W) * LDW + c];
            G[(idx / W) * LDW + c] = g;
            if (c >= N && c < 2 * N) pz += g * g;
          }
          gsync<NWG>(grp);
        } else {
        // reciprocal pivots off the dependent chain (independent divisions)
        double rr[M];
#pragma unroll
        for (int i = 0; i < M; ++i) rr[i] = 1.0 / rdiag[i];
        for (int c = gt; c < W; c += NT) {
          double x[M];
  #pragma unroll
          for (int i = M - 1; i >= 0; --i) {
            double v = H[i * LDW + c];
  #pragma unroll
            for (int k = i + 1; k < M; ++k) v -= Rm[i * ldr + k] * x[k];
            x[i] = v * rr[i];
          }
  #pragma unroll
          for (int i = 0; i < M; ++i) G[i * LDW + c] = -x[i];
          if (c >= N && c < 2 * N) {
  #pragma unroll
            for (int i = 0; i < M; ++i) pz += x[i] * x[i];
          }
        }
        gsync<NWG>(grp);
        }
        // one group reduction for both certificates (BIG: ||R||_F done above)
        double kz2;
        if constexpr (S::BIG) {
          kz2 = gsum<NWG>(pz, red, grp, gw);
        } else {
          const double2 t = gsum2<NWG>(pf, pz, red, grp, gw);
          rf2 = t.x;
          kz2 = t.y;
        }
        gsync<NWG>(grp);
        if (!S::BIG && sqrt(rf2) <= thr) {
          // p = 0: the gains come from the Cholesky branch below (G is
          // recomputed), all r rows stay (rotated by the QR: same row space)
          chol = true;
        } else if (!(kz2 * thr * thr < 1.0)) {
          status = PLQ_STATUS_RANK_REPAIR;
          if (s > 0) {
            mbar_wait(bar, phase);
            phase ^= 1u;
          }
          break;
        } else {
        // the surviving rows Q2' stack are rows M..r-1: advance the row base
        // instead of moving them (H is re-based at every segment start and
        // r + offset never exceeds the N-row buffer)
        H += M * LDW;
        r -= M;
        }
      }
    }
    PLQ_PHASE(4);   // constrained tail stage (QR, gains, rank certificate)
    if (chol) {
      // ---- G = -Muu^{-1} P (unconstrained stage, or p = 0), Cholesky in every lane's registers
      if (s > 0 && !constrained) stage_issue_group<N, M, NT>(p, st - 1, sm, bar, gt);
      if constexpr (S::BIG) {
        // CTA Cholesky of Muu in place (not needed again in this stage) and
        // a blocked DMMA solve of the m x W right-hand side
#ifdef PLQ_PHASE_PROFILE
        int nsync = 0;   // gchol8 syncs alternate: diagonal factor + panel | trailing tiles
        auto sy = [&] {
          gsync<NWG>(grp);
          if (nsync++ & 1)
            PLQ_PHASE(11);
          else
            PLQ_PHASE(15);
        };
#else
        auto sy = [&] { gsync<NWG>(grp); };
#endif
        static_assert(M * M >= 256 + NWG * 64, "TAU slot too small for the blocked solve");
        // Cholesky with the forward solve fused in: G <- L^{-1} (-P), block
        // row k in step k (no copy / negation passes)
        // Measured and rejected: a look-ahead variant (warp 0 factoring the
        // next diagonal block inside the trailing phase: slower, register
        // spills); gains through the explicit inverse (L^{-1} by an identity
        // right-hand side, Muu^{-1} = L^{-T} L^{-1}, G = -Muu^{-1} P as
        // parallel DMMA products: 8% faster, but K moved by ~1e-6 relative on
        // the cfg4-shape goldens -- cond(Muu)^2 error growth -- against ~1e-12
        // with the triangular solves)
        if (!gchol8<NWG>(Muu, M, LDM, tau, reinterpret_cast<int*>(sm + S::FLAG), gt, sy, nullptr, G, W, LDW,
                         tau + 256, P, -1.0)) {
          status = 1 + s;
          if (s > 0) {
            mbar_wait(bar, phase);
            phase ^= 1u;
          }
          break;
        }
        PLQ_PHASE(9);   // Cholesky + fused forward solve
        gtrsm8<1, NWG>(Muu, M, LDM, tau, G, W, LDW, tau + 256, gt, sy);   // G = -Muu^{-1} P
      } else {
      double Lr[M][M], id[M];
      int fail = 0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
#pragma unroll
        for (int i = k; i < M; ++i) {
          double v = Muu[i * LDM + k];
#pragma unroll
          for (int q = 0; q < k; ++q) v -= Lr[i][q] * Lr[k][q];
          if (i == k) {
            fail |= !(v > 0.0);
            const double vv = v > 0.0 ? v : 1.0;
            const double rs = rsqrt(vv);
            Lr[k][k] = vv * rs;
            id[k] = rs;
          } else {
            Lr[i][k] = v * id[k];
          }
        }
      }
      PLQ_PHASE(9);   // register Cholesky
      if (fail) {
        status = 1 + s;
        if (s > 0) {   // drain the copy in flight so the barrier phase stays in step
          mbar_wait(bar, phase);
          phase ^= 1u;
        }
        break;
      }
      for (int c = gt; c < W; c += NT) {
        double x[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          double v = P[i * LDW + c];
#pragma unroll
          for (int k = 0; k < i; ++k) v -= Lr[i][k] * x[k];
          x[i] = v * id[i];
        }
#pragma unroll
        for (int i = M - 1; i >= 0; --i) {
          double v = x[i];
#pragma unroll
          for (int k = i + 1; k < M; ++k) v -= Lr[k][i] * x[k];
          x[i] = v * id[i];
        }
#pragma unroll
        for (int i = 0; i < M; ++i) G[i * LDW + c] = -x[i];
      }
      gsync<NWG>(grp);
      }
    }

    PLQ_PHASE(5);   // Cholesky gains
    // ---- policy outputs
    for (int idx = gt; idx < M * N; idx += NT) {
      const int u = idx / N, c = idx % N;
      a.Kx[st * (M * N) + idx] = G[u * LDW + c];
      a.Kz[st * (M * N) + idx] = SERIAL ? 0.0 : G[u * LDW + N + c];
    }
    for (int u = gt; u < M; u += NT) a.k1[st * M + u] = G[u * LDW + CC];
    PLQ_PHASE(6);   // policy stores

    // ---- value update.  Tail stages: Y = P + Muu G, V += P'G + G'Y (the
    // reference's terms, endpoint.py:285-294).  Unconstrained stages have
    // G = -Muu^{-1} P, so Y = 0 in exact arithmetic and the update is the
    // standard Riccati form V += P'G (K = m instead of 2m, no Y GEMM).
    auto vupd = [&](int i, int c, double acc) {
      const int zi = i - N;
      double* d = (i < N) ? ((c < N) ? Vxx + i * LDN + c : dum)
                          : ((c < N) ? Vzx + zi * LDN + c : Vzz + zi * LDN + (c - N));
      *d += acc;
    };
    // SEL: the lower triangles of Vxx (mirrored: V is exactly symmetric, no
    // symmetrization pass) and Vzz (mirrored at the segment end), Vzx in
    // full, no wasted Vxz block; warp gw takes bands gw and TM-1-gw.
    constexpr int VTM = (N + NZ) / 8;
    auto vband = [](int w, int slot) { return slot == 0 ? w : (VTM > NWG ? VTM - 1 - w : -1); };
    auto von = [](int tm, int tn) { return tm < XB ? tn <= tm : (tn < XB || tn - XB <= tm - XB); };
    // Vzz (global scratch when BIG) is read before the k-loop (its latency
    // hides behind the DMMAs) and written back as pre + acc
    // (so are the on-chip Vxx / Vzx entries: no read-modify-write in the
    // epilogue); epi gets V + update
    auto vzero = [&](int i, int c) {
      if (i < N) return c <= i ? Vxx[i * LDN + c] : 0.0;
      const int zi = i - N;
      return c < N ? Vzx[zi * LDN + c] : (c - N <= zi ? Vzz[zi * LDN + (c - N)] : 0.0);
    };
    auto vsel = [&](int i, int c, double v) {
      if (i < N) {
        if (c <= i) {
          Vxx[i * LDN + c] = v;
          Vxx[c * LDN + i] = v;
        }
      } else {
        const int zi = i - N;
        if (c < N)
          Vzx[zi * LDN + c] = v;
        else if (c - N <= zi)
          Vzz[zi * LDN + (c - N)] = v;
      }
    };
    // SEL epilogue of the joint-band update: Vxx / Vzx read-modify-written
    // on chip, Vzz (L2 scratch) pre-loaded before the k-loop (has_pre)
    auto vsel2 = [&](int i, int c, double v, bool has_pre) {
      if (i < N) {
        if (c <= i) {
          const double w = Vxx[i * LDN + c] + v;
          Vxx[i * LDN + c] = w;
          Vxx[c * LDN + i] = w;
        }
      } else {
        const int zi = i - N;
        if (c < N)
          Vzx[zi * LDN + c] += v;
        else if (c - N <= zi)
          Vzz[zi * LDN + (c - N)] = has_pre ? v : Vzz[zi * LDN + (c - N)] + v;
      }
    };
    auto vzz_pre = [&](int i, int c) { return Vzz[(i - N) * LDN + (c - N)]; };
    if (constrained) {
      ggemm<M, W, M, false, LDM, LDW, NWG>(Muu, G, gw,
                                           [&](int i, int c, double acc) { Y[i * LDW + c] = P[i * LDW + c] + acc; });
      gsync<NWG>(grp);
      auto aP = [&](int i, int k) { return k < M ? P[k * LDW + i] : G[(k - M) * LDW + i]; };
      auto bG = [&](int k, int c) { return k < M ? G[k * LDW + c] : Y[(k - M) * LDW + c]; };
      if constexpr (SEL) {
        auto vu = [&](auto w) {
          constexpr int WI = decltype(w)::value;
          ggemm_sel2<N + NZ, W - 1, 2 * M, XB, 2 * XB, false, XB, WI, (VTM > NWG ? VTM - 1 - WI : -1)>(
              aP, bG, von, vzz_pre, vsel2);
        };
        warp_dispatch8(gw, vu);
      } else
        ggemm_f<N + NZ, W - 1, 2 * M, NWG>(aP, bG, gw, vupd);
    } else if constexpr (SEL) {
      auto vu = [&](auto w) {
        constexpr int WI = decltype(w)::value;
        ggemm_sel2<N + NZ, W - 1, M, XB, 2 * XB, false, XB, WI, (VTM > NWG ? VTM - 1 - WI : -1)>(
            [&](int i, int k) { return P[k * LDW + i]; }, [&](int k, int c) { return G[k * LDW + c]; }, von,
            vzz_pre, vsel2);
      };
      warp_dispatch8(gw, vu);
      PLQ_PHASE(13);   // value-update k-loops (warp 0's bands)
    } else {
      ggemm<N + NZ, W - 1, M, true, LDW, LDW, NWG>(P, G, gw, vupd);
    }
    // constant column (vx1, vz1) lane-parallel
    if (gt < N + NZ) {
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < M; ++u) t += P[u * LDW + gt] * G[u * LDW + CC];
      if (constrained) {
#pragma unroll
        for (int u = 0; u < M; ++u) t += G[u * LDW + gt] * Y[u * LDW + CC];
      }
      if (gt < N)
        vx1[gt] += t;
      else
        vz1[gt - N] += t;
    }
    gsync<NWG>(grp);
    PLQ_PHASE(7);   // value update
    if constexpr (!SEL) {
      // symmetrize Vxx (and Vzz) as 0.5 (V + V'): all N(N-1)/2 pairs in parallel
      // (Vzz is never a GEMM operand; symmetrizing it once per segment is the
      // same linear map as every stage: sym(sym(A) + X) = sym(A + X).)
      for (int pp = gt; pp < NP; pp += NT) {
        const int pr = pairs[pp];
        const int i = pr >> 8, c = pr & 255;
        const double v = 0.5 * (Vxx[i * LDN + c] + Vxx[c * LDN + i]);
        Vxx[i * LDN + c] = v;
        Vxx[c * LDN + i] = v;
      }
      gsync<NWG>(grp);
    }
  }
  if (!SERIAL) {
    for (int pp = gt; pp < NP; pp += NT) {
      const int pr = pairs[pp];
      const int i = pr >> 8, c = pr & 255;
      // SEL: only the lower triangle (c < i) was updated -- mirror it
      const double w = SEL ? Vzz[c * LDN + i] : 0.5 * (Vzz[i * LDN + c] + Vzz[c * LDN + i]);
      Vzz[i * LDN + c] = w;
      Vzz[c * LDN + i] = w;
    }
    gsync<NWG>(grp);
  }
  (void)lane;

  const int vsz = 3 * NN + 2 * N;
  if (a.vf0) {
    double* dst = a.vf0 + (b * J + j) * (int64_t)vsz;
    for (int idx = gt; idx < 3 * NN; idx += NT) {
      const int blk = idx / NN, e = idx % NN;
      const double* srcb = blk == 0 ? Vxx : (blk == 1 ? Vzx : Vzz);
      dst[idx] = srcb[(e / N) * LDN + e % N];
    }
    for (int i = gt; i < 2 * N; i += NT) dst[3 * NN + i] = sm[S::VX1 + i];
  }
  if (!SERIAL && r > 0 && status == 0 && a.feas) {
    // feasibility rows [Hx | Hz | h1] left at the segment start (parallel.py:452-456)
    double* dst = a.feas + (b * J + j) * (int64_t)N * (2 * N + 1);
    for (int idx = gt; idx < r * (2 * N + 1); idx += NT) {
      const int i = idx / (2 * N + 1), c = idx % (2 * N + 1);
      dst[idx] = H[i * LDW + c];
    }
  }
  if (gt == 0) {
    if (a.feas_rows) a.feas_rows[b * J + j] = (!SERIAL && status == 0) ? r : 0;
    if (status == 0 && !SERIAL && r > 0 && !a.feas) status = PLQ_STATUS_DEGENERATE;
    a.status[b * J + j] = status;
    if (status == PLQ_STATUS_RANK_REPAIR) push_repair(a, b, j);
  }
  gsync<NWG>(grp);
}

template <int N, int M, int NWG, int GROUPS>
__global__ void __launch_bounds__(NWG * 32 * GROUPS, (NWG == 1 ? 16 : 1)) sweep_small_kernel(SweepArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int grp = threadIdx.x / (NWG * 32);
  const int gt = threadIdx.x % (NWG * 32);
  double* sm = smem + grp * SL<N, M>::TOTAL;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SL<N, M>::BAR);
  // (i, c) pairs of the strict upper triangle, for the symmetrization
  __shared__ unsigned short pairs[N * (N - 1) / 2];
  for (int p = threadIdx.x; p < N * N; p += blockDim.x) {
    const int i = p / N, c = p % N;
    if (i < c) pairs[i * (2 * N - i - 1) / 2 + (c - i - 1)] = (unsigned short)((i << 8) | c);
  }
  __shared__ long long next_task[GROUPS];
  if (gt == 0) mbar_init(bar, 1 + NWG * 32);   // the bulk-copy arrive + every thread's cp.async arrive
  __syncthreads();
  uint32_t phase = 0;
  const int nloc = a.seg_end - a.seg_begin;
  const int64_t total = a.p.B * nloc;
  const int64_t first_free = (int64_t)gridDim.x * GROUPS;
  // first task static, the rest from a dynamic queue: segments differ in
  // cost (tail stages, serial last segment), so the tail of the launch
  // balances instead of following a fixed stride
  int64_t task = (int64_t)blockIdx.x * GROUPS + grp;
  while (task < total) {
    const int64_t b = task / nloc;
    const int j = a.seg_begin + (int)(task % nloc);
    if (!segment_bounds_ok(a.p, j)) {
      if (gt == 0) a.status[b * a.p.J + j] = PLQ_STATUS_BAD_PARTITION;
    } else if ((j == a.p.J - 1 && !a.endpoint_terminal) || a.smooth_vf0) {
      small_segment<N, M, NWG, true>(a, sm, grp, gt, b, j, phase, pairs);
    } else {
      small_segment<N, M, NWG, false>(a, sm, grp, gt, b, j, phase, pairs);
    }
    if (gt == 0)
      next_task[grp] = a.task_ctr ? first_free + (long long)atomicAdd(a.task_ctr, 1ULL) : task + first_free;
    gsync<NWG>(grp);
    task = next_task[grp];
    gsync<NWG>(grp);
  }
}

template <int N, int M, int NWG, int GROUPS>
int launch_small(const SweepArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(double) * SL<N, M>::TOTAL * GROUPS;
  auto kern = sweep_small_kernel<N, M, NWG, GROUPS>;
  static int per_sm = -1, sms = 148;
  static unsigned attr = 0;
  if (first_on_device(&attr)) {
    int dev = 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NWG * 32 * GROUPS, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tasks = a.p.B * (int64_t)(a.seg_end - a.seg_begin);
  SweepArgs args = a;
  // dynamic queue for the multi-warp groups (long tasks); the single-warp
  // n = 12 tasks are short enough that the queue round trip costs more
  if (NWG == 1) args.task_ctr = nullptr;
  if (args.task_ctr && cudaMemsetAsync(args.task_ctr, 0, sizeof(unsigned long long), s) != cudaSuccess) return -1;
  const int64_t blocks_needed = (tasks + GROUPS - 1) / GROUPS;
  const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(blocks_needed < cap ? blocks_needed : cap);
  kern<<<grid, NWG * 32 * GROUPS, smem, s>>>(args);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace

bool sweep_small_supported(int n, int m) {
  return (n == 12 && m == 4) || (n == 32 && m == 8) || (n == 64 && m == 32);
}

size_t sweep_small_gscratch_doubles(int n, int m) {
  if (n == 64 && m == 32) return (size_t)SL<64, 32>::GTOTAL;
  return 0;
}

int launch_sweep_small(const SweepArgs& a, cudaStream_t s) {
  if (a.p.n == 12 && a.p.m == 4) return launch_small<12, 4, 1, 1>(a, s);
  if (a.p.n == 32 && a.p.m == 8) return launch_small<32, 8, 4, 1>(a, s);
  if (a.p.n == 64 && a.p.m == 32) return launch_small<64, 32, 8, 1>(a, s);
  return -1;
}

#ifdef PLQ_PHASE_PROFILE
// copy (and reset) the per-CTA phase cycle counters: out[1024 * 16]
int sweep_small_phase_cycles(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles)) != cudaSuccess) return -1;
  static unsigned long long zero[1024][16];
  return cudaMemcpyToSymbol(g_phase_cycles, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;
}
#endif

}  // namespace plq
