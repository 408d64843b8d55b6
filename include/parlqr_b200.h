/*
 * parlqr_b200 -- C ABI of the B200-native horizon-partitioned Riccati solve.
 *
 * Drop-in for the hot path of the reference package `parlqr`
 * (/root/reference/pkg/src/parlqr), whose Python entry point is
 *
 *     parlqr.solve_parallel(problem, J, workers=None, tolerances=...,
 *                           collect_diagnostics=False, partition=None)
 *                                                    (parallel.py:422-553)
 *
 * Plain pointers and sizes only; no torch types.  All arrays are float64,
 * row-major, C-contiguous, in the reference's stacked transport layout
 * (`_stacked_stages`, parallel.py:108,141-149) with a leading batch axis B.
 * The library never allocates device memory persistently: callers size the
 * workspace with plq_workspace_bytes() and own every buffer.
 */
#ifndef PARLQR_B200_H
#define PARLQR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLQ_ABI_VERSION 2

/* Return codes of the entry points (launch / argument errors only; numerical
 * failures are reported per segment in plq_outputs_t.status). */
#define PLQ_OK 0
#define PLQ_ERR_ARG (-1)         /* invalid argument (shapes, null pointers, partition) */
#define PLQ_ERR_CUDA (-2)        /* a CUDA launch or copy failed; see plq_last_error() */
#define PLQ_ERR_WORKSPACE (-3)   /* workspace smaller than plq_workspace_bytes() */

/* Per-(problem, segment) status values, mapped to the reference exceptions
 * by the Python host layer (errors.py:8-51):
 *   0          ok
 *   1 + t      CholeskyFailure(t), t = segment-local stage (endpoint.py:243-245,
 *              serial.py:63-66)
 *   -1         segment ends with feasibility rows (a degenerate partition,
 *              parallel.py:322-384, 452-456) but plq_outputs_t.feas is NULL, so
 *              the constrained link solve cannot run -> UnsupportedPartition
 *   -2         LinkSingular (parallel.py:267-271); stored in segment 0's slot
 *   -3         Infeasible(residual, segment) (parallel.py:462-475)
 *   -4         malformed partition (ValueError, parallel.py:88-89, 434-440) */
#define PLQ_STATUS_OK 0
#define PLQ_STATUS_DEGENERATE (-1)
#define PLQ_STATUS_LINK_SINGULAR (-2)
#define PLQ_STATUS_INFEASIBLE (-3)  /* segment's feasibility rows violated at the solved links */
#define PLQ_STATUS_BAD_PARTITION (-4) /* split_times not increasing from 0 to T, or a segment longer
                                         than max_seg_len (checked on the device; the segment is
                                         skipped, the Python layer raises ValueError) */

/* One batch of B independent problems sharing (T, n, m) and one partition.
 * Replaces the (problem, partition, tolerances) arguments of
 * parlqr.solve_parallel (parallel.py:422-445).  Device pointers. */
typedef struct plq_problem {
  int64_t B;                 /* problems in the batch */
  int32_t T, n, m, J;        /* horizon, state dim, control dim, segments (1 <= J <= T) */
  int32_t max_seg_len;       /* max(split_times[j+1]-split_times[j]) */
  const int32_t* split_times;/* J+1 increasing stage indices, 0 .. T (Partition.split_times) */
  const double* Qxx;         /* (B,T,n,n) symmetric -- PRECONDITION: Qxx, Quu, QxxT must be exactly
                                symmetric, as the reference's constructors make them (problem.py:106-116);
                                some kernels read one triangle only.  The Python layer symmetrizes. */
  const double* Qux;         /* (B,T,m,n) */
  const double* Quu;         /* (B,T,m,m) symmetric */
  const double* qx1;         /* (B,T,n) */
  const double* qu1;         /* (B,T,m) */
  const double* Fx;          /* (B,T,n,n) */
  const double* Fu;          /* (B,T,n,m) */
  const double* f1;          /* (B,T,n) */
  const double* QxxT;        /* (B,n,n) terminal Qxx (TerminalCost) */
  const double* qx1T;        /* (B,n) terminal qx1 */
  const double* x_init;      /* (B,n) */
  double rank_tol;           /* ToleranceSet.rank_tol (problem.py:53) */
  double feas_tol;           /* ToleranceSet.feas_tol (problem.py:54) */
} plq_problem_t;

/* Caller-allocated device outputs of one solve (LqrSolution + ParallelDetails,
 * problem.py:262-280, parallel.py:390-405). */
typedef struct plq_outputs {
  double* K;              /* (B,T,m,n)  policies[t].Kx */
  double* k;              /* (B,T,m)    policies[t].k1 (folded k = Kz z + k1) */
  double* x;              /* (B,T+1,n)  states */
  double* u;              /* (B,T,m)    controls */
  double* lam;            /* (B,T+1,n)  lambdas */
  double* links;          /* (B,J-1,n)  details.link_points */
  double* mu_left;        /* (B,J-1,n)  details.mu_left */
  double* lambda_right;   /* (B,J-1,n)  details.lambda_right */
  double* vf0;            /* (B,J,3n^2+2n) details.segment_values0: Vxx0,Vzx0,Vzz0,vx10,vz10
                             (the last, serial segment fills Vxx0 and vx10 only) */
  double* Kz;             /* (B,T,m,n)  unfolded segment gains (_solve_segment_task "Kz"); may be NULL */
  double* k1;             /* (B,T,m)    unfolded segment offsets ("k1"); may be NULL */
  double* objective;      /* (B) */
  double* kkt_inf;        /* (B) kkt_residual_inf */
  double* link_mismatch;  /* (B) details.link_mismatch */
  double* link_residual;  /* (B) details.link_residual */
  int32_t* status;        /* (B,J) see PLQ_STATUS_* */
  /* Degenerate partitions (segments that cannot reach arbitrary endpoints,
   * parallel.py:320-384, 452-475).  All three NULL: such segments report
   * PLQ_STATUS_DEGENERATE.  Given: the rows are returned and the links come
   * from the feasibility-constrained dense KKT solve. */
  double* feas;           /* (B,J,n,2n+1) details.segment_feasibility rows [Hx | Hz | h1] (an orthonormal
                             rotation of the reference's rows; row counts in feas_rows) */
  int32_t* feas_rows;     /* (B,J) */
  double* feas_residual;  /* (B,J) details.feasibility_residuals */
  /* collect_diagnostics=True (StageDiagnostics, endpoint.py:108-115, 258-299).  Both NULL: not
   * collected.  Given: every endpoint segment is solved by the rank-revealing kernel (SVD of the
   * triangular factor of Nu, csrc/plq_rank.cuh) and reports the worst defects over its constrained
   * stages: [0] basis_defect = |V V' - I|_max of the right singular basis [Py | Zw], [1]
   * projector_defect = |P P - P|_max of the row projector P = I - U_p U_p' (both in the
   * QR-rotated coordinates of that kernel); diag_rows = max_rows, the largest constraint-to-go row
   * count.  The last (serial) segment has no diagnostics (zeros; the reference returns None).
   * Not copied back by plq_solve_parallel_host. */
  double* diag;           /* (B,J,2) */
  int32_t* diag_rows;     /* (B,J) */
} plq_outputs_t;

/* Library identification. */
int plq_abi_version(void);
const char* plq_last_error(void);

/* Workspace for plq_solve_parallel (and the phase entry points below). */
size_t plq_workspace_bytes(const plq_problem_t* problem);

/* Full partitioned solve of every problem in the batch, stream-ordered:
 * segment sweeps (replaces _run_tasks/_solve_segment_task, parallel.py:197-240,
 * endpoint.backward_pass endpoint.py:168-301, serial.backward_pass
 * serial.py:37-79), link solve (assemble_link_system + LinkSystem.solve,
 * parallel.py:264-319, endpoint.py:410-438), reconstruction
 * (parallel.py:478-527) and diagnostics (evaluate_objective, kkt_residual,
 * problem.py:366-420).  `stream` is a cudaStream_t (NULL = legacy default). */
int plq_solve_parallel(const plq_problem_t* problem, const plq_outputs_t* out, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Same solve from HOST buffers (the end-to-end entry a ctypes/cgo binding of
 * the reference would call): `host_problem` holds host pointers in every
 * array field (split_times included), `host_out` host destinations (any may
 * be NULL to skip the copy back).  Copies in, solves, copies out, returns
 * after the stream is synchronized.  `device_arena` must hold
 * plq_host_arena_bytes() bytes of device memory. */
size_t plq_host_arena_bytes(const plq_problem_t* host_problem);
int plq_solve_parallel_host(const plq_problem_t* host_problem, const plq_outputs_t* host_out, void* device_arena,
                            size_t arena_bytes, void* stream);

/* Phase entry points for horizon sharding across GPUs (one process per GPU;
 * the caller exchanges data between phases, e.g. NCCL all-gathers).  The
 * same `workspace` must be passed to every phase of one solve.
 *   1. plq_sweep_segments: sweeps of segments [seg_begin, seg_end) of every
 *      problem -> out->K, Kz/k1 (workspace if NULL), vf0, status.
 *      [exchange: vf0 rows of all segments]
 *   2. plq_link_solve: replicated coupling solve from the complete vf0
 *      -> links, link_residual, status (LinkSingular).
 *   3. plq_reconstruct_segments: fold, rollout, multipliers, per-segment
 *      objective / interior-KKT partials for [seg_begin, seg_end) -> k, x, u,
 *      lam, mu_left, lambda_right, partials[b][j][0..1].
 *      [exchange: mu_left, lambda_right]
 *   4. plq_boundary_segments: KKT rows of the link stages of [seg_begin,
 *      seg_end) (need the right neighbour's lambda) -> partials[b][j][2].
 *      [exchange: partials]
 *   5. plq_finalize: fixed-order reduction of the complete `partials`
 *      (B,J,3) into objective, kkt_inf and link_mismatch. */
int plq_sweep_segments(const plq_problem_t* problem, const plq_outputs_t* out, int32_t seg_begin, int32_t seg_end,
                       void* workspace, size_t workspace_bytes, void* stream);
int plq_link_solve(const plq_problem_t* problem, const plq_outputs_t* out, void* workspace, size_t workspace_bytes,
                   void* stream);
int plq_reconstruct_segments(const plq_problem_t* problem, const plq_outputs_t* out, int32_t seg_begin,
                             int32_t seg_end, double* partials, void* workspace, size_t workspace_bytes, void* stream);
int plq_boundary_segments(const plq_problem_t* problem, const plq_outputs_t* out, int32_t seg_begin,
                          int32_t seg_end, double* partials, void* workspace, size_t workspace_bytes, void* stream);
int plq_finalize(const plq_problem_t* problem, const plq_outputs_t* out, const double* partials, void* workspace,
                 size_t workspace_bytes, void* stream);

/* Horizon-sharded solve across the ranks of an NCCL communicator (one process
 * per GPU): the five phases above with their three exchanges issued by the
 * library on `stream` -- no host synchronization, no allocation.  Replaces the
 * reference's worker pool over segments (_run_tasks, parallel.py:168-207,
 * 446-449) for horizons too long for one GPU's latency budget (cfg2, cfg3).
 *   * rank r sweeps / reconstructs the balanced contiguous segment range
 *     [r*(J/nranks) + min(r, J%nranks), ...) (remainder to the early ranks);
 *     it reads only its own segments' stages, so `problem`'s stage arrays may
 *     hold just that window (pointers shifted back by the window's first
 *     stage); QxxT, qx1T, x_init are replicated.
 *   * exchanges (in place, on the full-size output arrays every rank holds):
 *     vf0 + status (+ feas, feas_rows when given) rows after the sweeps;
 *     mu_left / lambda_right rows after the reconstruction; the (B,J,3)
 *     partials before the fixed-order reduction.  Equal shards of one problem
 *     travel as one in-place ncclAllGather per array, anything else as grouped
 *     in-place ncclBroadcast calls.  The link solve is replicated, so links,
 *     objective, kkt_inf, link_mismatch, status are bitwise identical on every
 *     rank and identical for any rank count.
 *   * K, k, x, u, lam hold this rank's segments only (the caller gathers them
 *     if it wants the whole trajectory in one place).
 * `nccl_comm` is an ncclComm_t whose rank/size are `rank`/`nranks` (NULL is
 * allowed for nranks == 1: the phases run without NCCL).  NCCL is bound at run
 * time with dlopen("libnccl.so.2") (override: PLQ_NCCL_LIB); this library has
 * no link-time NCCL dependency. */
int plq_solve_parallel_sharded(const plq_problem_t* problem, const plq_outputs_t* out, void* workspace,
                               size_t workspace_bytes, void* nccl_comm, int32_t rank, int32_t nranks, void* stream);

/* Device-side seeded generator of the benchmark inputs (
 * the reference generates its benchmark problems on the host, bench.py:38-60
 * via generate.py:14-47, and BASELINE.json gives the recipe used here): fills
 * the ARRAYS NAMED BY `problem` (device pointers; they are outputs of this
 * call, split_times / J / max_seg_len are ignored) with problems
 * first_problem .. first_problem + B - 1 of the seeded family
 *   Fx = I + a_scale G/sqrt(n), Fu = 0.1 Bu/sqrt(n), f1 = 0.1 c,
 *   Qxx = W W'/n + q_eps I, Quu = V V'/m + r_eps I, Qux = 0, qx1, qu1 ~ N(0,1),
 *   QxxT = WT WT'/n + q_eps I, qx1T, x_init ~ N(0,1)
 * (all capitals / lowercase letters independent N(0,1) arrays; Qxx, Quu, QxxT
 * exactly symmetric).  Counter-based (Philox-4x32-10 + Box-Muller, stream
 * documented in csrc/plq_generate.cu): the values depend only on (seed,
 * problem index, field, element), so a batch generated in pieces equals one
 * generated in one call. */
typedef struct plq_recipe {
  double a_scale, q_eps, r_eps;
  uint64_t seed;
  int64_t first_problem;
} plq_recipe_t;
int plq_generate_batch(const plq_problem_t* problem, const plq_recipe_t* recipe, void* stream);

/* Device outputs of the smoothing pass (parlqr.parallel.smooth,
 * parallel.py:567-633): the smoothed LqrSolution's policies, trajectory and
 * diagnostics.  Its lambdas are the parent's (unchanged). */
typedef struct plq_smooth_outputs {
  double* K;              /* (B,T,m,n) smoothed policies[t].Kx (parent's on the last segment) */
  double* k;              /* (B,T,m)   smoothed policies[t].k1 */
  double* x;              /* (B,T+1,n) states of the rollout of those policies from x_init */
  double* u;              /* (B,T,m)   controls */
  double* objective;      /* (B) evaluate_objective(states, controls) */
  double* kkt_inf;        /* (B) kkt_residual with the parent's lambdas */
  double* deviation;      /* (B) details.smooth_deviation = max |x - x_parent|, |u - u_parent| */
  int32_t* status;        /* (B,J) 1+t: CholeskyFailure(t) in the sweep of segment j, else 0 */
} plq_smooth_outputs_t;

/* Smoothing pass over the completed parallel solve `parent` of the same
 * problem batch (reads parent->K, k, x, u, lam, links, vf0): the sweeps of
 * segments 0..J-2 with terminal cost TerminalCost(Vxx0_{j+1}, vx10_{j+1} +
 * Vzx0_{j+1}' z_{j+1}) (serial.backward_pass, serial.py:37-79), then one
 * rollout of all T policies (_rollout_policies, parallel.py:556-564) fused
 * with the objective / KKT / deviation of the result.  The workspace is the
 * plq_workspace_bytes() one.  J = 1 reproduces the parent (smooth() returns
 * it unchanged, parallel.py:587-589). */
int plq_smooth(const plq_problem_t* problem, const plq_outputs_t* parent, const plq_smooth_outputs_t* out,
               void* workspace, size_t workspace_bytes, void* stream);

/* Two-point-boundary solve (parlqr.endpoint.solve_endpoint_affine /
 * solve_endpoint, endpoint.py:603-653) of every problem in the batch:
 * problem->J must be 1 (split_times = {0, T}).  W = 2n+1.
 * Device outputs of plq_endpoint_affine: */
typedef struct plq_endpoint_outputs {
  double* Kx;             /* (B,T,m,n)  policies[t].Kx */
  double* Kz;             /* (B,T,m,n)  policies[t].Kz */
  double* k1;             /* (B,T,m)    policies[t].k1 */
  double* value0;         /* (B,3n^2+2n) values[0]: Vxx, Vzx, Vzz, vx1, vz1 */
  double* X;              /* (B,T+1,n,W) maps: x_t = [Ra|Rz|r1] [x_init; x_term; 1] */
  double* S;              /* (B,T,m,W)   maps: u_t = [Sa|Sz|s1] [...] */
  double* Lam;            /* (B,T+1,n,W) multipliers: lam_t = [La|Lz|l1] [...] */
  double* E;              /* (B,n,W)     mu = [Ea|Ez|e1] [...] */
  int32_t* status;        /* (B) backward pass: 0, 1+t CholeskyFailure(t), -1 unreachable endpoint
                             directions (feasibility rows) when feas / feas_rows are NULL */
  int32_t* gram_status;   /* (B) multiplier Gram system: 0, 1+i FactorizationFailure(block i), or -1 = not
                             computed (feasibility rows: the boundary constraints are linearly dependent,
                             solve_endpoint_affine endpoint.py:589-620 leaves multipliers = None) */
  /* Unreachable endpoint directions (T m < n, or no control authority): the rows [Hx | Hz | h1] any
   * (x_init, x_term) pair must satisfy (BackwardResult.feasibility, endpoint.py:124-127; an orthonormal
   * rotation of the reference's rows).  Both NULL: such problems report status -1. */
  double* feas;           /* (B,n,W) */
  int32_t* feas_rows;     /* (B) */
  /* collect_diagnostics=True (as plq_outputs_t::diag / diag_rows): both NULL = not collected */
  double* diag;           /* (B,2) basis / projector defects */
  int32_t* diag_rows;     /* (B) max_rows */
} plq_endpoint_outputs_t;

/* Evaluation at concrete endpoints (EndpointAffineSolution.evaluate,
 * endpoint.py:538-575): trajectories, objective and the full KKT stack. */
typedef struct plq_endpoint_point {
  const double* x_init;   /* (B,n) device; NULL = problem->x_init */
  const double* x_term;   /* (B,n) device */
  double* x;              /* (B,T+1,n) */
  double* u;              /* (B,T,m) */
  double* lam;            /* (B,T+1,n) */
  double* mu;             /* (B,n) */
  double* objective;      /* (B) */
  double* kkt_inf;        /* (B) */
  double* feas_residual;  /* (B) max |Hx x_init + Hz x_term + h1| over the feasibility rows (0 without rows);
                             may be NULL.  The caller raises Infeasible above feas_tol * scale
                             (endpoint.py:516-523).  Problems with rows take their multipliers from the
                             value-function gradient and the stationarity recursion (gradient_duals,
                             endpoint.py:566-587). */
} plq_endpoint_point_t;

size_t plq_endpoint_workspace_bytes(const plq_problem_t* problem);
/* backward_pass(stages, terminal) (endpoint.py:168-301), forward_pass
 * (:326-349), multiplier_pass (:452-476). */
int plq_endpoint_affine(const plq_problem_t* problem, const plq_endpoint_outputs_t* out, void* workspace,
                        size_t workspace_bytes, void* stream);
int plq_endpoint_evaluate(const plq_problem_t* problem, const plq_endpoint_outputs_t* affine,
                          const plq_endpoint_point_t* point, void* workspace, size_t workspace_bytes, void* stream);

/* Number of kernel launches the last plq_solve_parallel / phase call issued
 * on this thread (evidence for bench.py's gpu_launches). */
int plq_last_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* PARLQR_B200_H */
