// Internal (non-ABI) declarations shared by the kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/parlqr_b200.h"

namespace plq {

// One-time per-device setup guard: kernel attributes (dynamic shared memory
// opt-in, carveout) are per device, so a process driving several GPUs must
// set them on each.  `mask` is a function-local static bitmask.
inline bool first_on_device(unsigned* mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned bit = 1u << (dev & 31);
  if (*mask & bit) return false;
  *mask |= bit;
  return true;
}

// Per-CTA scratch buffers of the segment sweep.  Each one is placed in
// shared memory or in a per-CTA slice of global scratch by plan_sweep().
enum SweepBuf {
  SB_V = 0,   // [Vxx; Vzx; Vzz] (3n x n) then vx1 (n), vz1 (n)
  SB_IN,      // stage inputs: F=[Fx|Fu|f1] (n x (n+m+1)), Qxx, Qux, Quu, qx1, qu1
  SB_PGY,     // P, G, Y (each m x W, W = 2n+1)
  SB_MUU,     // Muu (m x m) then its Cholesky factor (m x m)
  SB_MISC,    // tau (m), rdiag (m), reduction scratch (32), flags
  SB_VF,      // Vxx*F (n x (n+m+1)); reused as the N = Hx*F temp in tail stages
  SB_Z,       // Vzx*F (n x (n+m+1)) = [Mzx | Mzu | Vzx f1 + vz1]
  SB_MX,      // [Mxx | mx1] (n x (n+1))
  SB_H,       // constraint rows [Hx | Hz | h1] (n x W)
  SB_WIDE,    // mixed-branch scratch (only when n % m != 0)
  SB_COUNT
};

// stages of the tiled GEMM's cp.async ring in the large-mode sweep.  Measured
// on the cfg3 sweep (B200): 2 stages 13.0 ms, 4 stages 13.3 ms -- the deeper
// ring's shared memory comes out of the L1 the panel / epilogue loads use, and
// the GEMM k-loops were not waiting on their copies.
constexpr int sweep_tile_stages(int threads) { return threads == 256 ? 2 : 2; }

// large mode, blocked factorizations, m <= 64: the Cholesky of Muu runs on a
// shared-memory copy (m x (m + 4) doubles behind the MISC scratch) instead of
// the L2-resident scratch -- its 8 block steps are latency chains
__host__ __device__ inline bool sweep_muu_in_smem(int n, int m) { return n >= 48 && m >= 16 && m <= 64; }

struct SweepLayout {
  int64_t off[SB_COUNT];     // offset in doubles within its space
  int in_smem[SB_COUNT];
  int64_t smem_doubles;
  int64_t gmem_doubles;      // per CTA
  int large;                 // n >= 48: buffers in global scratch, smem holds GEMM tiles
  int64_t tiles_off;         // smem offset of the tiled-GEMM staging area
};

// Segment j of the partition is well formed: 1 <= L <= max_seg_len, the
// first segment starts at 0 and the last ends at T.  The kernels whose
// shared-memory buffers are sized from max_seg_len skip (and the sweeps
// flag, PLQ_STATUS_BAD_PARTITION) a segment that is not -- the C ABI cannot
// read device-resident split_times without a host synchronization.
__host__ __device__ inline bool segment_bounds_ok(const plq_problem_t& p, int j) {
  const int lo = p.split_times[j], hi = p.split_times[j + 1];
  return hi - lo >= 1 && hi - lo <= p.max_seg_len && (j > 0 || lo == 0) && (j < p.J - 1 || hi == p.T);
}

struct SweepArgs {
  plq_problem_t p;
  double* Kx;      // (B,T,m,n)
  double* Kz;      // (B,T,m,n)
  double* k1;      // (B,T,m)
  double* vf0;     // (B,J,3n^2+2n)
  int32_t* status; // (B,J)
  double* gscratch;
  SweepLayout lay;
  int seg_begin, seg_end;  // segment range [seg_begin, seg_end) of every problem
  // Smoothing pass (parallel.py:567-633): when set, every swept segment is a
  // plain (serial) sweep whose terminal cost is segment j+1's start value
  // conditioned on its link point; vf0 may then be null (not written).
  const double* smooth_vf0;    // (B,J,3n^2+2n) parent solve's start values
  const double* smooth_links;  // (B,J-1,n) parent solve's link points
  // Two-point-boundary solve (endpoint.backward_pass(stages, terminal),
  // endpoint.py:168-301 as called by solve_endpoint[_affine]): the last
  // segment is an endpoint sweep seeded with the terminal cost.
  int endpoint_terminal;
  // degenerate partitions: rows left at a segment start are written here
  // (else the segment reports PLQ_STATUS_DEGENERATE)
  double* feas;          // (B,J,n,2n+1)
  int32_t* feas_rows;    // (B,J)
  // dynamic task queue of the specialized sweep (reset by the launcher);
  // null: static round-robin
  unsigned long long* task_ctr;
  // Rank-revealing repair (plq_rank.cuh): a sweep that cannot certify the
  // rank of a tail stage's Nu marks the segment PLQ_STATUS_RANK_REPAIR and
  // appends b*J+j to repair_list; the repair launch of the generic kernel
  // (repair = 1) re-solves exactly those segments with the SVD decision,
  // using rank_scratch (rank_scratch_doubles per CTA).  The counter is reset
  // before every sweep.
  int repair;
  unsigned long long* repair_ctr;
  long long* repair_list;      // (B*J)
  double* rank_scratch;
  int64_t rank_scratch_doubles;
  // collect_diagnostics (StageDiagnostics, endpoint.py:108-115): force_repair
  // sends every endpoint segment to the repair launch, which has the singular
  // vectors and writes the defects / row counts here
  int force_repair;
  double* diag;          // (B,J,2)
  int32_t* diag_rows;    // (B,J)
};

// internal status: segment awaits the rank-revealing repair pass (never
// returned to the caller: the repair pass overwrites it)
#define PLQ_STATUS_RANK_REPAIR (-5)

__device__ __forceinline__ void push_repair(const SweepArgs& a, int64_t b, int j) {
  if (!a.repair && a.repair_ctr) {
    const unsigned long long i = atomicAdd(a.repair_ctr, 1ULL);
    a.repair_list[i] = (long long)(b * a.p.J + j);
  }
}

struct LinkFeasArgs {
  plq_problem_t p;
  const double* vf0;
  const double* feas;
  const int32_t* feas_rows;
  double* links;
  double* link_residual;
  double* mu_corr;       // (B,J,n) Hz' nu per segment
  double* feas_residual; // (B,J)
  int32_t* status;
  double* pool;          // dense KKT scratch when it exceeds shared memory
  int dmax;
};
int link_feas_dmax(int J, int n);
size_t link_feas_pool_doubles(int64_t B, int J, int n);
int launch_link_feas(const LinkFeasArgs& a, cudaStream_t s);

// Device-side terminal cost of a swept segment: the problem's terminal cost
// for the last segment, or -- in the smoothing pass -- TerminalCost(Vxx,
// vx1 + Vzx' z) of segment j+1 (TerminalCost symmetrizes, problem.py:129-133).
struct SmoothArgs {
  plq_problem_t p;
  const double* K0;    // parent policies (B,T,m,n), (B,T,m)
  const double* k0;
  const double* x0;    // parent states / controls / multipliers
  const double* u0;
  const double* lam0;
  double* K;           // smoothed policies: sweeps wrote stages < split[J-1]
  double* k;
  double* x;           // (B,T+1,n)
  double* u;           // (B,T,m)
  double* objective;   // (B,)
  double* kkt;         // (B,)
  double* deviation;   // (B,)
  double* maps;        // segmented mode: (B,J-1,n,n+1) closed-loop segment maps [Phi | c],
                       // then (B,J) join residuals and (B,ceil(T/CH),3) evaluation partials
};

constexpr int SMOOTH_EVAL_CH = 8;   // stages per evaluation CTA (segmented mode)
size_t smooth_map_doubles(int64_t B, int T, int J, int n, int m);

// Segment-parallel rollout (affine segment maps) when the batch alone cannot
// fill the GPU; otherwise one CTA walks each problem's horizon.
bool smooth_segmented(int64_t B, int J);
int launch_smooth_rollout(const SmoothArgs& a, cudaStream_t s, int* launches);

// Two-point-boundary solve (plq_endpoint.cu)
size_t endpoint_scratch_doubles(const plq_problem_t& p);
size_t endpoint_eval_doubles(const plq_problem_t& p);
int launch_endpoint_maps_mult(const plq_problem_t& p, const plq_endpoint_outputs_t& o, double* ws, cudaStream_t s,
                              int* launches);
int launch_endpoint_evaluate(const plq_problem_t& p, const plq_endpoint_outputs_t& o, const plq_endpoint_point_t& pt,
                             double* ws, cudaStream_t s, int* launches);

struct ReconArgs {
  plq_problem_t p;
  const double* Kx;
  const double* Kz;
  const double* k1;
  const double* vf0;
  const double* links;   // (B,J-1,n)
  double* k;             // (B,T,m)
  double* x;             // (B,T+1,n)
  double* u;             // (B,T,m)
  double* lam;           // (B,T+1,n)
  double* mu_left;       // (B,J-1,n)
  double* lambda_right;  // (B,J-1,n)
  double* gh;            // (B,T,n+m) per-stage g = Qxx x + Qux' u + qx1, h = Qux x + Quu u + qu1
  double* xend;          // (B,J,n) rollout end state of each segment
  double* part;          // (B,J,3) objective partial, interior KKT, link-stage KKT
  int seg_begin, seg_end;
  const double* mu_corr; // (B,J,n) Hz' nu of degenerate segments (parallel.py:511-513), or null
  const int32_t* feas_rows;  // (B,J): mu_corr is valid where > 0
};

int launch_sweep(const SweepArgs& a, int grid, int threads, size_t smem, cudaStream_t s);
int sweep_threads(int n);
int sweep_max_blocks_per_sm(int threads, size_t smem);
SweepLayout plan_sweep(int n, int m, int threads, size_t smem_budget);

int launch_recon(const ReconArgs& a, cudaStream_t s);
int launch_boundary(const ReconArgs& a, double* bpart, cudaStream_t s);
int launch_finalize(const plq_problem_t& p, const double* part, const double* bpart, const double* mu_left,
                    const double* lambda_right, const double* link_res, double* objective, double* kkt,
                    double* mismatch, double* link_residual, cudaStream_t s);

// Specialized small-state kernels (compile-time n, m).
bool sweep_small_supported(int n, int m);
size_t sweep_small_gscratch_doubles(int n, int m);   // per CTA (n >= 64 variants)
int launch_sweep_small(const SweepArgs& a, cudaStream_t s);
bool recon_small_supported(int n, int m);
bool recon_split_supported(int n, int m);
int launch_recon_split(const ReconArgs& a, cudaStream_t s);
int launch_recon_small(const ReconArgs& a, cudaStream_t s);
bool link_seq_supported(int n, int J);
size_t link_seq_workspace_doubles(int64_t B, int J, int n);
int launch_link_seq(const plq_problem_t& p, const double* vf0, double* links, double* link_residual,
                    int32_t* status, double* ws, cudaStream_t s);

// Device-side seeded generator of the BASELINE recipe (plq_generate.cu).
int launch_generate(const plq_problem_t& p, double a_scale, double q_eps, double r_eps, uint64_t seed, int64_t first,
                    cudaStream_t s);

// Link solve of a batch of short chains, one CTA per problem (plq_linkchain.cu).
bool link_chain_supported(int n, int J);
bool link_chain_preferred(int64_t B, int J);
size_t link_chain_workspace_doubles(int64_t B, int J, int n);
int launch_link_chain(const plq_problem_t& p, const double* vf0, double* links, double* link_residual,
                      int32_t* status, double* ws, cudaStream_t s);

// Link (coupling) solve by block cyclic reduction.
size_t link_workspace_doubles(int64_t B, int J, int n);
int launch_link_solve(const plq_problem_t& p, const double* vf0, double* links, double* link_residual,
                      int32_t* status, double* ws, cudaStream_t s, int* launches);

}  // namespace plq
