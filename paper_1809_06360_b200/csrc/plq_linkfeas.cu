// Link solve for partitions with reachability-deficient segments
// (_solve_links_with_feasibility, parallel.py:320-384) and the feasibility
// check at the solved links (parallel.py:462-475).
//
// A problem whose endpoint segments left feasibility rows (Hx, Hz, h1) --
// segments too short to reach arbitrary endpoints -- minimizes the summed
// segment cost-to-go over the links subject to every segment's rows: the
// dense KKT system over [links; nu] (dimension (J-1) n + sum r_j), assembled
// exactly as the reference does and solved by LU with partial pivoting (the
// reference's np.linalg.solve), one CTA per problem.  The rows the GPU
// sweeps emit are an orthonormal rotation of the reference's SVD-compressed
// rows, which leaves the links and the multiplier correction Hz' nu
// unchanged.  Outputs per problem: links, link_residual = 0 (as the
// reference reports), mu_corr[j] = Hz_j' nu_j (subtracted from mu_j by the
// reconstruction, parallel.py:511-513), the per-segment feasibility residual
// and PLQ_STATUS_INFEASIBLE where it exceeds feas_tol * scale * 10.
// Problems without rows are only tested (256 per pass); mu_corr is read by
// the reconstruction only where a segment has rows.
#include <cuda_runtime.h>

#include "plq_device.cuh"
#include "plq_internal.h"

namespace plq {
namespace {

constexpr int LF_NT = 256;
constexpr size_t LF_SMEM = 160 * 1024;

__global__ void __launch_bounds__(LF_NT) link_feas_kernel(LinkFeasArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double rv[LF_NT / 32];
  __shared__ int ri[LF_NT / 32];
  __shared__ int piv_s;
  __shared__ int bad_s;
  const plq_problem_t& p = a.p;
  const int n = p.n, J = p.J, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NN = n * n, VS = 3 * NN + 2 * n, W = 2 * n + 1;
  const int nl = (J - 1) * n;
  __shared__ int list[LF_NT];
  __shared__ int cnt;
  // 256 problems per pass: one thread per problem tests for rows, only the
  // degenerate ones are solved (mu_corr is read only where rows exist)
  for (int64_t base = (int64_t)blockIdx.x * LF_NT; base < p.B; base += (int64_t)gridDim.x * LF_NT) {
    if (tid == 0) cnt = 0;
    __syncthreads();
    if (J >= 128) {
      // long chains (few problems): a warp sums one problem's row counts
      for (int q = warp; q < LF_NT && base + q < p.B; q += LF_NT / 32) {
        int R = 0;
        for (int j = lane; j < J; j += 32) R += a.feas_rows[(base + q) * J + j];
        R = __reduce_add_sync(0xffffffffu, R);
        if (lane == 0 && R > 0) list[atomicAdd(&cnt, 1)] = q;
      }
    } else {
      const int64_t bt = base + tid;
      int R = 0;
      if (bt < p.B)
        for (int j = 0; j < J; ++j) R += a.feas_rows[bt * J + j];
      if (R > 0) list[atomicAdd(&cnt, 1)] = tid;
    }
    __syncthreads();
    const int count = cnt;
  for (int li = 0; li < count; ++li) {
    const int64_t b = base + list[li];
    const int32_t* rows = a.feas_rows + b * J;
    int R = 0;
    for (int j = 0; j < J; ++j) R += rows[j];
    const int dim = nl + R;
    if (dim > a.dmax) {   // too large for the dense path: unsupported
      if (tid == 0) a.status[b * J] = PLQ_STATUS_DEGENERATE;
      continue;
    }
    double* A = ((size_t)dim * (dim + 1) * sizeof(double) <= LF_SMEM) ? sm
                                                                       : a.pool + (int64_t)blockIdx.x * a.dmax * (a.dmax + 1);
    double* bb = A + (int64_t)dim * dim;
    const double* xi = p.x_init + b * n;
    const double* vf = a.vf0 + b * (int64_t)J * VS;
    for (int idx = tid; idx < dim * (dim + 1); idx += LF_NT) A[idx] = 0.0;
    __syncthreads();
    // link blocks (parallel.py:341-363): row block k-1 of link k = 1..J-1
    for (int idx = tid; idx < (J - 1) * NN; idx += LF_NT) {
      const int k = 1 + idx / NN, r = (idx % NN) / n, c = idx % n;
      const double* left = vf + (k - 1) * VS;
      const double* right = vf + k * VS;
      const int row = (k - 1) * n + r;
      A[(int64_t)row * dim + (k - 1) * n + c] = left[2 * NN + r * n + c] + right[r * n + c];
      if (k > 1) A[(int64_t)row * dim + (k - 2) * n + c] = left[NN + r * n + c];
      if (k < J - 1) A[(int64_t)row * dim + k * n + c] = right[NN + c * n + r];
    }
    for (int idx = tid; idx < (J - 1) * n; idx += LF_NT) {
      const int k = 1 + idx / n, r = idx % n;
      const double* left = vf + (k - 1) * VS;
      const double* right = vf + k * VS;
      double v = -left[3 * NN + n + r];
      if (k == 1) {
        double t = 0.0;
        for (int c = 0; c < n; ++c) t += left[NN + r * n + c] * xi[c];
        v -= t;
      }
      bb[(k - 1) * n + r] = v - right[3 * NN + r];
    }
    // feasibility rows (parallel.py:364-377)
    int off = nl;
    for (int j = 0; j < J; ++j) {
      const int rj = rows[j];
      if (!rj) continue;
      const double* H = a.feas + (b * J + j) * (int64_t)n * W;
      for (int idx = tid; idx < rj * n; idx += LF_NT) {
        const int i = idx / n, c = idx % n;
        const double hz = H[i * W + n + c];
        A[(int64_t)(off + i) * dim + j * n + c] = hz;
        A[(int64_t)(j * n + c) * dim + off + i] = hz;
        if (j > 0) {
          const double hx = H[i * W + c];
          A[(int64_t)(off + i) * dim + (j - 1) * n + c] = hx;
          A[(int64_t)((j - 1) * n + c) * dim + off + i] = hx;
        }
      }
      for (int i = tid; i < rj; i += LF_NT) {
        double v = -H[i * W + 2 * n];
        if (j == 0) {
          double t = 0.0;
          for (int c = 0; c < n; ++c) t += H[i * W + c] * xi[c];
          v -= t;
        }
        bb[off + i] = v;
      }
      off += rj;
    }
    if (tid == 0) bad_s = 0;
    __syncthreads();
    // LU with partial pivoting (LAPACK getrf: first index of max |a_ik|)
    for (int k = 0; k < dim; ++k) {
      double best = -1.0;
      int bi = k;
      for (int i = k + tid; i < dim; i += LF_NT) {
        const double v = fabs(A[(int64_t)i * dim + k]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        rv[warp] = best;
        ri[warp] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double bv = rv[0];
        int bx = ri[0];
        for (int w = 1; w < LF_NT / 32; ++w)
          if (rv[w] > bv || (rv[w] == bv && ri[w] < bx)) {
            bv = rv[w];
            bx = ri[w];
          }
        piv_s = bx;
        if (!(bv > 0.0)) bad_s = 1;
      }
      __syncthreads();
      if (bad_s) break;
      const int pv = piv_s;
      if (pv != k) {
        for (int c = tid; c <= dim; c += LF_NT) {
          double* r0 = (c < dim) ? A + (int64_t)k * dim + c : bb + k;
          double* r1 = (c < dim) ? A + (int64_t)pv * dim + c : bb + pv;
          const double t = *r0;
          *r0 = *r1;
          *r1 = t;
        }
        __syncthreads();
      }
      const double rinv = 1.0 / A[(int64_t)k * dim + k];
      for (int i = k + 1 + tid; i < dim; i += LF_NT) A[(int64_t)i * dim + k] *= rinv;
      __syncthreads();
      const int s = dim - k - 1;
      for (int idx = tid; idx < s * s; idx += LF_NT) {
        const int i = k + 1 + idx / s, c = k + 1 + idx % s;
        A[(int64_t)i * dim + c] -= A[(int64_t)i * dim + k] * A[(int64_t)k * dim + c];
      }
      __syncthreads();
    }
    if (bad_s) {
      if (tid == 0 && (a.status[b * J] == 0 || a.status[b * J] == PLQ_STATUS_LINK_SINGULAR))
        a.status[b * J] = PLQ_STATUS_LINK_SINGULAR;
      __syncthreads();
      continue;
    }
    // L y = P b, then U x = y
    for (int k = 0; k < dim; ++k) {
      const double yk = bb[k];
      for (int i = k + 1 + tid; i < dim; i += LF_NT) bb[i] -= A[(int64_t)i * dim + k] * yk;
      __syncthreads();
    }
    for (int k = dim - 1; k >= 0; --k) {
      if (tid == 0) bb[k] /= A[(int64_t)k * dim + k];
      __syncthreads();
      const double xk = bb[k];
      for (int i = tid; i < k; i += LF_NT) bb[i] -= A[(int64_t)i * dim + k] * xk;
      __syncthreads();
    }
    // links, the regular link solve's verdict replaced, mu corrections
    for (int idx = tid; idx < nl; idx += LF_NT) a.links[b * nl + idx] = bb[idx];
    if (tid == 0) {
      a.link_residual[b] = 0.0;
      if (a.status[b * J] == PLQ_STATUS_LINK_SINGULAR) a.status[b * J] = 0;
    }
    __syncthreads();
    off = nl;
    for (int j = 0; j < J; ++j) {
      const int rj = rows[j];
      if (!rj) continue;
      const double* H = a.feas + (b * J + j) * (int64_t)n * W;
      for (int c = tid; c < n; c += LF_NT) {
        double t = 0.0;
        for (int i = 0; i < rj; ++i) t += H[i * W + n + c] * bb[off + i];
        a.mu_corr[(b * J + j) * n + c] = t;
      }
      // feasibility residual at the solved links (parallel.py:462-475)
      const double* av = (j == 0) ? xi : bb + (j - 1) * n;
      const double* zv = bb + j * n;
      double worst = 0.0, amax = 0.0, zmax = 0.0;
      for (int i = tid; i < rj; i += LF_NT) {
        double t = H[i * W + 2 * n];
        for (int c = 0; c < n; ++c) t += H[i * W + c] * av[c] + H[i * W + n + c] * zv[c];
        worst = fmax(worst, fabs(t));
      }
      for (int c = tid; c < n; c += LF_NT) {
        amax = fmax(amax, fabs(av[c]));
        zmax = fmax(zmax, fabs(zv[c]));
      }
      worst = block_max(worst, rv);
      amax = block_max(amax, rv);
      zmax = block_max(zmax, rv);
      if (tid == 0) {
        a.feas_residual[b * J + j] = worst;
        if (worst > p.feas_tol * (1.0 + amax + zmax) * 10.0 && a.status[b * J + j] == 0)
          a.status[b * J + j] = PLQ_STATUS_INFEASIBLE;
      }
      __syncthreads();
      off += rj;
    }
  }
    __syncthreads();
  }
}

}  // namespace

int link_feas_dmax(int J, int n) {
  const int64_t d = 2LL * (J - 1) * n;
  return (int)(d < 1024 ? d : 1024);
}

size_t link_feas_pool_doubles(int64_t B, int J, int n) {
  const int64_t d = link_feas_dmax(J, n);
  if ((size_t)d * (d + 1) * sizeof(double) <= LF_SMEM) return 0;
  const int64_t ctas = B < 32 ? B : 32;
  return (size_t)ctas * d * (d + 1);
}

int launch_link_feas(const LinkFeasArgs& args, cudaStream_t s) {
  LinkFeasArgs a = args;
  a.dmax = link_feas_dmax(a.p.J, a.p.n);
  static unsigned attr = 0;
  if (first_on_device(&attr))
    cudaFuncSetAttribute(link_feas_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LF_SMEM);
  const int64_t chunks = (a.p.B + LF_NT - 1) / LF_NT;
  const int grid = (int)(chunks < 32 ? chunks : 32);
  link_feas_kernel<<<grid, LF_NT, LF_SMEM, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace plq
