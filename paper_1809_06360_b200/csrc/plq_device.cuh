// CTA-level fp64 building blocks for the partitioned Riccati kernels (sm_100a).
//
// All matrices are row-major with an explicit leading dimension.  Pointers
// are generic: a buffer may live in shared memory or in a per-CTA slice of
// global scratch (L2-resident) -- the host-side layout decides which, so one
// kernel body serves n = 1 .. 128.
//
// GEMMs run on the FP64 tensor pipe through warp-level `mma.sync.m8n8k4.f64`
// (SASS DMMA.8x8x4).  On B200 DMMA and DFMA have the same peak (measured
// 37.0 TFLOP/s, tools/fp64_peak.cu); DMMA wins by needing one shared-memory
// operand load per 256 multiply-adds instead of one per 2-4.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace plq {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `red` needs blockDim/32 doubles of scratch.  All threads
// receive the result.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = red[0];
  for (int w = 1; w < nw; ++w) t = fmax(t, red[w]);
  return t;
}

// C(MxN) = op(A)(MxK) * op(B)(KxN), delivered element-wise to `epi(i, j, acc)`.
// TA: A is stored transposed (A(i,k) = A[k*lda+i]); TB likewise for B.
// Each warp owns (8*BM)x(8*BN) output super-tiles; out-of-range operand
// elements read as zero so ragged shapes need no padding.
template <bool TA, bool TB, int BM, int BN, class Epi>
__device__ __forceinline__ void cta_gemm(int M, int N, int K, const double* __restrict__ A, int lda,
                                         const double* __restrict__ B, int ldb, Epi epi) {
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

// In-place lower Cholesky of the m x m SPD block A (lower triangle used and
// overwritten; the strict upper triangle is left untouched).  Returns false
// on a non-positive (or NaN) pivot, the LAPACK dpotrf failure condition that
// numpy.linalg.cholesky reports as LinAlgError.
//
// Right-looking with the unscaled pivot column, A_ij -= A_ik A_jk / A_kk
// (rows by warp, columns by lane: one barrier per column, no index division);
// the columns are scaled by 1/sqrt(pivot) in one pass at the end.  Every
// thread reads the same pivot, so the failure exit is uniform.
__device__ __forceinline__ bool cta_cholesky(double* A, int m, int lda, int* /*flag*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  for (int k = 0; k < m; ++k) {
    const double dkk = A[k * lda + k];
    if (!(dkk > 0.0)) return false;
    const double inv = 1.0 / dkk;
    for (int i = k + 1 + warp; i < m; i += nw) {
      const double aik = A[i * lda + k] * inv;
      for (int j = k + 1 + lane; j <= i; j += 32) A[i * lda + j] -= aik * A[j * lda + k];
    }
    __syncthreads();
  }
  // off-diagonal entries first (they read the unscaled pivots), then the diagonal
  for (int i = warp; i < m; i += nw)
    for (int k = lane; k < i; k += 32) A[i * lda + k] /= sqrt(A[k * lda + k]);
  __syncthreads();
  for (int k = threadIdx.x; k < m; k += blockDim.x) A[k * lda + k] = sqrt(A[k * lda + k]);
  __syncthreads();
  return true;
}

// X <- (L L')^{-1} X for the m x W right-hand side X (cho_solve), thread per column.
__device__ __forceinline__ void cta_cho_solve(const double* L, int m, int ldl, double* X, int W, int ldx) {
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    for (int i = 0; i < m; ++i) {
      double s = X[i * ldx + c];
      for (int k = 0; k < i; ++k) s -= L[i * ldl + k] * X[k * ldx + c];
      X[i * ldx + c] = s / L[i * ldl + i];
    }
    for (int i = m - 1; i >= 0; --i) {
      double s = X[i * ldx + c];
      for (int k = i + 1; k < m; ++k) s -= L[k * ldl + i] * X[k * ldx + c];
      X[i * ldx + c] = s / L[i * ldl + i];
    }
  }
  __syncthreads();
}

// X <- L^{-1} X (forward substitution only), thread per column.
__device__ __forceinline__ void cta_trsm_lower(const double* L, int m, int ldl, double* X, int W, int ldx) {
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    for (int i = 0; i < m; ++i) {
      double s = X[i * ldx + c];
      for (int k = 0; k < i; ++k) s -= L[i * ldl + k] * X[k * ldx + c];
      X[i * ldx + c] = s / L[i * ldl + i];
    }
  }
  __syncthreads();
}

// Householder QR of the r x m panel A (r >= m), applied on the left to the
// r x W block X as well.  On exit the upper triangle of A holds R, the
// reflector tails sit below the diagonal and X holds Q' X.  `rdiag` gets the
// m diagonal entries of R.  Column j's reflector is H_j = I - tau v v' with
// v_j = 1, chosen so R_jj = -sign(a_jj) ||a_j:r,j|| (LAPACK dlarfg).
__device__ __forceinline__ void cta_householder_qr(double* A, int r, int m, int lda, double* X, int W, int ldx,
                                                   double* tau, double* rdiag, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int j = 0; j < m; ++j) {
    double part = 0.0;
    for (int i = j + 1 + tid; i < r; i += nt) {
      const double v = A[i * lda + j];
      part += v * v;
    }
    const double sig = block_sum(part, red);
    const double alpha = A[j * lda + j];
    double t = 0.0, beta = alpha, scale = 0.0;
    if (sig > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + sig), alpha);
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < r; i += nt) A[i * lda + j] *= scale;
    if (tid == 0) {
      tau[j] = t;
      rdiag[j] = beta;
    }
    __syncthreads();
    // apply H_j to the trailing columns of A and to all columns of X
    const int ncols = (m - j - 1) + W;
    for (int c = tid; c < ncols; c += nt) {
      double* col;
      int ld;
      if (c < m - j - 1) {
        col = A + (j + 1 + c);
        ld = lda;
      } else {
        col = X + (c - (m - j - 1));
        ld = ldx;
      }
      double s = col[j * ld];
      for (int i = j + 1; i < r; ++i) s += A[i * lda + j] * col[i * ld];
      s *= t;
      col[j * ld] -= s;
      for (int i = j + 1; i < r; ++i) col[i * ld] -= s * A[i * lda + j];
    }
    __syncthreads();
    if (tid == 0) A[j * lda + j] = beta;
    __syncthreads();
  }
}

// Apply the reflectors stored in A (from cta_householder_qr with `p`
// reflectors over `r` rows) to the r x W block X:  X <- Q X (reverse=true)
// or X <- Q' X (reverse=false).
__device__ __forceinline__ void cta_apply_q(const double* A, int r, int p, int lda, const double* tau, double* X,
                                            int W, int ldx, bool reverse) {
  for (int step = 0; step < p; ++step) {
    const int j = reverse ? (p - 1 - step) : step;
    const double t = tau[j];
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
      double s = X[j * ldx + c];
      for (int i = j + 1; i < r; ++i) s += A[i * lda + j] * X[i * ldx + c];
      s *= t;
      X[j * ldx + c] -= s;
      for (int i = j + 1; i < r; ++i) X[i * ldx + c] -= s * A[i * lda + j];
    }
    __syncthreads();
  }
}

// y = op(A) x for an R x C matrix A (op(A) = A' when TA), thread per output.
template <bool TA>
__device__ __forceinline__ void cta_matvec(int R, int C, const double* A, int lda, const double* x, double* y,
                                           double alpha, const double* add) {
  const int rows = TA ? C : R, inner = TA ? R : C;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < inner; ++k) s += (TA ? A[k * lda + i] : A[i * lda + k]) * x[k];
    y[i] = alpha * s + (add ? add[i] : 0.0);
  }
}

}  // namespace plq
