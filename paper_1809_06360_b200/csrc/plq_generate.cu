// Device-side seeded problem generator: the BASELINE.json
// synthetic recipe (the host restatement is synth.generate_one)
// written straight into the stacked (B,T,...) device layout of plq_problem_t, so
// a batch never exists on the host (cfg4: 28 GB).
//
// Per problem p (global index first_problem + b) and stage t:
//   Fx = I + a_scale G / sqrt(n),  Fu = 0.1 Bu / sqrt(n),  f1 = 0.1 c,
//   Qxx = W W'/n + q_eps I,  Quu = V V'/m + r_eps I,  Qux = 0,
//   qx1 = q,  qu1 = r;   terminal QxxT = WT WT'/n + q_eps I, qx1T, x_init,
// every capital / lowercase letter an independent N(0,1) array.
//
// Random stream (documented so that a host restatement can reproduce it,
// synth.device_stream_reference): Philox-4x32-10 with key = (seed lo, seed hi)
// and counter = (k lo, k hi, field id, problem index), where k = e >> 1 for the
// e-th element (row-major over (T, ...) within the problem) of the field; the
// four output words give two uniforms u = (hi >> 5) 2^-27 + (lo >> 6) 2^-53 and
// one Box-Muller pair  z0 = r cos(2 pi u1), z1 = r sin(2 pi u1),
// r = sqrt(-2 log(1 - u0));  element e takes z_{e & 1}.  The stream depends only
// on (seed, problem index, field, element), never on the launch shape: batches
// generated in pieces (first_problem offsets) are identical to one call.
// Qxx / Quu are computed on the lower triangle and mirrored, so they are
// exactly symmetric (the reference's constructors symmetrize, problem.py:106-116).
#include <math.h>
#include <stdint.h>

#include "plq_internal.h"

namespace plq {

namespace {

enum Field : uint32_t { F_G = 0, F_BU = 1, F_C = 2, F_W = 3, F_V = 4, F_Q = 5, F_R = 6, F_WT = 7, F_QT = 8, F_X0 = 9 };

__device__ __forceinline__ void philox_round(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
  const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
  const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
  const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
  c[0] = n0;
  c[1] = lo1;
  c[2] = n2;
  c[3] = lo0;
}

// standard normal number e of (seed, problem, field)
__device__ __forceinline__ double normal_at(uint64_t seed, uint32_t problem, uint32_t field, uint64_t e) {
  const uint64_t k = e >> 1;
  uint32_t c[4] = {(uint32_t)k, (uint32_t)(k >> 32), field, problem};
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const double u0 = (double)(c[0] >> 5) * (1.0 / 134217728.0) + (double)(c[1] >> 6) * (1.0 / 9007199254740992.0);
  const double u1 = (double)(c[2] >> 5) * (1.0 / 134217728.0) + (double)(c[3] >> 6) * (1.0 / 9007199254740992.0);
  const double r = sqrt(-2.0 * log(1.0 - u0));
  double sn, cs;
  sincospi(2.0 * u1, &sn, &cs);
  return (e & 1) ? r * sn : r * cs;
}

struct GenArgs {
  plq_problem_t p;   // array fields are the OUTPUTS
  double a_scale, q_eps, r_eps;
  uint64_t seed;
  int64_t first;
};

// A A'/d + eps I of the d x d block A (shared memory, stride ld), lower triangle
// computed and mirrored
__device__ __forceinline__ void gram_out(const double* A, int d, int ld, double eps, double* out) {
  const double inv = 1.0 / (double)d;
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int i = idx / d, j = idx % d;
    if (j > i) continue;
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc += A[i * ld + k] * A[j * ld + k];
    const double v = acc * inv + (i == j ? eps : 0.0);
    out[i * d + j] = v;
    out[j * d + i] = v;
  }
}

// one CTA per (problem, stage)
__global__ void __launch_bounds__(256) gen_stage_kernel(GenArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int n = a.p.n, m = a.p.m, T = a.p.T;
  const int64_t st = blockIdx.x;            // b * T + t
  const int64_t b = st / T, t = st % T;
  const uint32_t prob = (uint32_t)(a.first + b);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nn = n * n, nm = n * m, mm = m * m, ld = n + 1, ldm = m + 1;
  double* Fx = const_cast<double*>(a.p.Fx) + st * nn;
  double* Fu = const_cast<double*>(a.p.Fu) + st * nm;
  double* f1 = const_cast<double*>(a.p.f1) + st * n;
  double* Qxx = const_cast<double*>(a.p.Qxx) + st * nn;
  double* Qux = const_cast<double*>(a.p.Qux) + st * nm;
  double* Quu = const_cast<double*>(a.p.Quu) + st * mm;
  double* qx1 = const_cast<double*>(a.p.qx1) + st * n;
  double* qu1 = const_cast<double*>(a.p.qu1) + st * m;
  const double sa = a.a_scale / sqrt((double)n), sb = 0.1 / sqrt((double)n);
  for (int idx = tid; idx < nn; idx += nt) {
    Fx[idx] = (idx / n == idx % n ? 1.0 : 0.0) + sa * normal_at(a.seed, prob, F_G, (uint64_t)t * nn + idx);
    sm[(idx / n) * ld + idx % n] = normal_at(a.seed, prob, F_W, (uint64_t)t * nn + idx);
  }
  for (int idx = tid; idx < nm; idx += nt) {
    Fu[idx] = sb * normal_at(a.seed, prob, F_BU, (uint64_t)t * nm + idx);
    Qux[idx] = 0.0;
  }
  for (int i = tid; i < n; i += nt) {
    f1[i] = 0.1 * normal_at(a.seed, prob, F_C, (uint64_t)t * n + i);
    qx1[i] = normal_at(a.seed, prob, F_Q, (uint64_t)t * n + i);
  }
  for (int i = tid; i < m; i += nt) qu1[i] = normal_at(a.seed, prob, F_R, (uint64_t)t * m + i);
  double* Vs = sm + (size_t)n * ld;
  for (int idx = tid; idx < mm; idx += nt)
    Vs[(idx / m) * ldm + idx % m] = normal_at(a.seed, prob, F_V, (uint64_t)t * mm + idx);
  __syncthreads();
  gram_out(sm, n, ld, a.q_eps, Qxx);
  gram_out(Vs, m, ldm, a.r_eps, Quu);
}

// one CTA per problem: terminal cost and initial state
__global__ void __launch_bounds__(256) gen_terminal_kernel(GenArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int n = a.p.n, nn = n * n, ld = n + 1;
  const int64_t b = blockIdx.x;
  const uint32_t prob = (uint32_t)(a.first + b);
  for (int idx = threadIdx.x; idx < nn; idx += blockDim.x)
    sm[(idx / n) * ld + idx % n] = normal_at(a.seed, prob, F_WT, (uint64_t)idx);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const_cast<double*>(a.p.qx1T)[b * n + i] = normal_at(a.seed, prob, F_QT, (uint64_t)i);
    const_cast<double*>(a.p.x_init)[b * n + i] = normal_at(a.seed, prob, F_X0, (uint64_t)i);
  }
  __syncthreads();
  gram_out(sm, n, ld, a.q_eps, const_cast<double*>(a.p.QxxT) + b * nn);
}

}  // namespace

int launch_generate(const plq_problem_t& p, double a_scale, double q_eps, double r_eps, uint64_t seed, int64_t first,
                    cudaStream_t s) {
  GenArgs a{p, a_scale, q_eps, r_eps, seed, first};
  const size_t sm_stage = sizeof(double) * ((size_t)p.n * (p.n + 1) + (size_t)p.m * (p.m + 1));
  const size_t sm_term = sizeof(double) * (size_t)p.n * (p.n + 1);
  if (sm_stage > 48 * 1024)
    cudaFuncSetAttribute(gen_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_stage);
  if (sm_term > 48 * 1024)
    cudaFuncSetAttribute(gen_terminal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_term);
  const int64_t stages = p.B * (int64_t)p.T;
  if (stages > 0x7fffffffLL) return -1;
  gen_stage_kernel<<<(unsigned)stages, 256, sm_stage, s>>>(a);
  gen_terminal_kernel<<<(unsigned)p.B, 256, sm_term, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace plq
