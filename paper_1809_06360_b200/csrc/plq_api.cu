// C-ABI layer (include/parlqr_b200.h): argument checks, workspace carving,
// and the stream-ordered phase sequence of one partitioned solve.
#include <dlfcn.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "plq_internal.h"
#include "plq_rank.cuh"

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

// PLQ_FORCE_GENERIC=1 routes every shape through the generic kernels (tests
// use it to keep the generic path covered on the config shapes).
bool force_generic() {
  const char* e = getenv("PLQ_FORCE_GENERIC");
  return e && e[0] == '1';
}
bool use_small_sweep(const plq_problem_t* p) { return !force_generic() && plq::sweep_small_supported(p->n, p->m); }
bool use_small_recon(const plq_problem_t* p) { return !force_generic() && plq::recon_small_supported(p->n, p->m); }
// PLQ_LINK=bcr forces block cyclic reduction for the link solve (measurement)
bool force_bcr() {
  const char* e = getenv("PLQ_LINK");
  return e && e[0] == 'b';
}
bool use_seq_link(const plq_problem_t* p) {
  return !force_generic() && !force_bcr() && plq::link_seq_supported(p->n, p->J);
}
// one CTA per problem running the reference's sequential block Cholesky
// (16 <= n <= 64): when the batch is at least as large as the chain is long,
// or forced with PLQ_LINK=chain
bool use_chain_link(const plq_problem_t* p) {
  if (force_generic() || force_bcr() || !plq::link_chain_supported(p->n, p->J)) return false;
  const char* e = getenv("PLQ_LINK");
  return (e && e[0] == 'c') || plq::link_chain_preferred(p->B, p->J);
}

int fail(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

int cuda_fail(const char* where) {
  const cudaError_t e = cudaGetLastError();
  snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return PLQ_ERR_CUDA;
}

inline size_t up2(size_t x) { return (x + 1) & ~size_t(1); }

struct Plan {
  plq::SweepLayout lay;
  int threads = 0;
  size_t smem = 0;
  int grid_max = 0;
  size_t off_Kz = 0, off_k1 = 0, off_gh = 0, off_xend = 0, off_part = 0, off_gs = 0, off_link = 0, off_smap = 0;
  size_t off_mucorr = 0, off_lfpool = 0, off_ctr = 0, off_rlist = 0, off_rank = 0;
  size_t rank_doubles = 0;   // per repair CTA
  int repair_grid = 0;
  size_t total_doubles = 0;
};

int check_problem(const plq_problem_t* p) {
  if (!p) return fail(PLQ_ERR_ARG, "null problem");
  if (p->B < 1 || p->T < 1 || p->n < 1 || p->m < 1) return fail(PLQ_ERR_ARG, "B, T, n, m must be >= 1");
  if (p->J < 1 || p->J > p->T) return fail(PLQ_ERR_ARG, "J must be in [1, T]");
  if (p->n > 128 || p->m > 128) return fail(PLQ_ERR_ARG, "n and m are limited to 128");
  if (p->max_seg_len < 1 || p->max_seg_len > p->T) return fail(PLQ_ERR_ARG, "bad max_seg_len");
  if (!p->split_times || !p->Qxx || !p->Qux || !p->Quu || !p->qx1 || !p->qu1 || !p->Fx || !p->Fu || !p->f1 ||
      !p->QxxT || !p->qx1T || !p->x_init)
    return fail(PLQ_ERR_ARG, "null problem array");
  return PLQ_OK;
}

Plan make_plan(const plq_problem_t* p) {
  Plan P;
  const int64_t B = p->B, T = p->T, n = p->n, m = p->m, J = p->J;
  P.threads = plq::sweep_threads(p->n);
  if (const char* e = getenv("PLQ_SWEEP_THREADS")) P.threads = atoi(e);   // measurement override
  const size_t budget = 200 * 1024;
  P.lay = plq::plan_sweep(p->n, p->m, P.threads, budget);
  P.smem = (size_t)P.lay.smem_doubles * sizeof(double);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = plq::sweep_max_blocks_per_sm(P.threads, P.smem);
  if (per_sm < 1) per_sm = 1;
  P.grid_max = sms * per_sm;
  size_t off = 0;
  P.off_Kz = off;
  off += up2(B * T * m * n);
  P.off_k1 = off;
  off += up2(B * T * m);
  P.off_gh = off;
  off += up2(B * T * (n + m));
  P.off_xend = off;
  off += up2(B * J * n);
  P.off_part = off;
  off += up2(B * J * 3);
  P.off_gs = off;
  off += up2(std::max((size_t)P.grid_max * P.lay.gmem_doubles,
                      (size_t)sms * 2 * plq::sweep_small_gscratch_doubles(p->n, p->m)));
  P.off_link = off;
  off += up2(std::max({plq::link_workspace_doubles(B, p->J, p->n),
                       use_seq_link(p) ? plq::link_seq_workspace_doubles(B, p->J, p->n) : size_t(0),
                       use_chain_link(p) ? plq::link_chain_workspace_doubles(B, p->J, p->n) : size_t(0)}));
  P.off_ctr = off;
  off += 2;   // [0] dynamic segment queue, [1] rank-repair count
  P.off_rlist = off;
  off += up2(B * J);   // rank-repair list (long long per entry)
  // rank-revealing repair launch (plq_rank.cuh): one resident wave of the
  // generic kernel at most, each CTA with its own slow-path scratch
  P.repair_grid = std::min(P.grid_max, sms);
  P.rank_doubles = up2(plq::rank_scratch_doubles(p->n, p->m, P.lay.large ? 2 * p->n + 2 : 2 * p->n + 1));
  P.off_rank = off;
  off += (size_t)P.repair_grid * P.rank_doubles;
  P.off_mucorr = off;
  off += up2(B * J * n);
  P.off_lfpool = off;
  if (J > 1) off += up2(plq::link_feas_pool_doubles(B, p->J, p->n));
  P.off_smap = off;
  if (plq::smooth_segmented(B, p->J)) off += up2(plq::smooth_map_doubles(B, p->T, p->J, p->n, p->m));
  P.total_doubles = off;
  return P;
}

struct Ctx {
  Plan P;
  double* ws;
  double* Kz;
  double* k1;
  cudaStream_t s;
};

int setup(const plq_problem_t* p, const plq_outputs_t* o, void* ws, size_t bytes, void* stream, Ctx* c) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (!o) return fail(PLQ_ERR_ARG, "null outputs");
  if (!ws) return fail(PLQ_ERR_ARG, "null workspace");
  c->P = make_plan(p);
  if (bytes < c->P.total_doubles * sizeof(double)) return fail(PLQ_ERR_WORKSPACE, "workspace too small");
  c->ws = static_cast<double*>(ws);
  c->Kz = o->Kz ? o->Kz : c->ws + c->P.off_Kz;
  c->k1 = o->k1 ? o->k1 : c->ws + c->P.off_k1;
  c->s = static_cast<cudaStream_t>(stream);
  return PLQ_OK;
}

int phase_sweep(const plq_problem_t* p, const plq_outputs_t* o, Ctx& c, int j0, int j1, int endpoint_terminal = 0) {
  if (!o->K || !o->vf0 || !o->status) return fail(PLQ_ERR_ARG, "null sweep output");
  if (j0 < 0 || j1 > p->J || j0 >= j1) return fail(PLQ_ERR_ARG, "bad segment range");
  plq::SweepArgs a{};
  a.p = *p;
  a.Kx = o->K;
  a.Kz = c.Kz;
  a.k1 = c.k1;
  a.vf0 = o->vf0;
  a.status = o->status;
  a.gscratch = c.ws + c.P.off_gs;
  a.task_ctr = reinterpret_cast<unsigned long long*>(c.ws + c.P.off_ctr);
  a.lay = c.P.lay;
  a.seg_begin = j0;
  a.seg_end = j1;
  a.endpoint_terminal = endpoint_terminal;
  a.feas = o->feas;
  a.feas_rows = o->feas_rows;
  a.repair_ctr = reinterpret_cast<unsigned long long*>(c.ws + c.P.off_ctr) + 1;
  a.repair_list = reinterpret_cast<long long*>(c.ws + c.P.off_rlist);
  a.rank_scratch = c.ws + c.P.off_rank;
  a.rank_scratch_doubles = (int64_t)c.P.rank_doubles;
  // collect_diagnostics: endpoint segments solved by the rank-revealing launch of the generic kernel
  if ((o->diag != nullptr) != (o->diag_rows != nullptr)) return fail(PLQ_ERR_ARG, "diag and diag_rows go together");
  const bool diag = o->diag != nullptr;
  a.force_repair = diag ? 1 : 0;
  a.diag = diag ? o->diag : nullptr;
  a.diag_rows = diag ? o->diag_rows : nullptr;
  if (diag) {
    const size_t cells = (size_t)p->B * p->J;
    if (cudaMemsetAsync(o->diag, 0, cells * 2 * sizeof(double), c.s) != cudaSuccess ||
        cudaMemsetAsync(o->diag_rows, 0, cells * sizeof(int32_t), c.s) != cudaSuccess)
      return cuda_fail("diagnostics reset");
  }
  // endpoint segments (tail stages) may need the rank-revealing repair pass
  const bool tails = endpoint_terminal || j0 < p->J - 1;
  if (tails && cudaMemsetAsync(a.repair_ctr, 0, sizeof(unsigned long long), c.s) != cudaSuccess)
    return cuda_fail("repair counter reset");
  const int64_t tasks = p->B * (int64_t)(j1 - j0);
  const int grid = (int)std::min<int64_t>(tasks, c.P.grid_max);
  const int rc = (use_small_sweep(p) && !diag) ? plq::launch_sweep_small(a, c.s)
                                               : plq::launch_sweep(a, grid, c.P.threads, c.P.smem, c.s);
  if (rc) return cuda_fail("sweep launch");
  ++g_launches;
  if (tails) {
    // re-solve (exact SVD rank decision) the segments whose tail-stage rank
    // the fast sweep could not certify; exits at once when there are none
    plq::SweepArgs ra = a;
    ra.repair = 1;
    if (plq::launch_sweep(ra, c.P.repair_grid, c.P.threads, c.P.smem, c.s)) return cuda_fail("rank repair launch");
    ++g_launches;
  }
  return PLQ_OK;
}

int phase_link(const plq_problem_t* p, const plq_outputs_t* o, Ctx& c) {
  if (!o->links || !o->link_residual || !o->vf0 || !o->status) return fail(PLQ_ERR_ARG, "null link output");
  int nl = 0;
  if (p->J < 2) return PLQ_OK;
  if (use_seq_link(p)) {
    if (plq::launch_link_seq(*p, o->vf0, o->links, o->link_residual, o->status, c.ws + c.P.off_link, c.s))
      return cuda_fail("link launch");
    nl = 1;
  } else if (use_chain_link(p)) {
    if (plq::launch_link_chain(*p, o->vf0, o->links, o->link_residual, o->status, c.ws + c.P.off_link, c.s))
      return cuda_fail("link launch");
    nl = 1;
  } else if (plq::launch_link_solve(*p, o->vf0, o->links, o->link_residual, o->status, c.ws + c.P.off_link, c.s,
                                    &nl)) {
    return cuda_fail("link launch");
  }
  if (o->feas && o->feas_rows && o->feas_residual) {
    // problems with feasibility rows: the constrained dense link solve replaces the links
    plq::LinkFeasArgs lf{};
    lf.p = *p;
    lf.vf0 = o->vf0;
    lf.feas = o->feas;
    lf.feas_rows = o->feas_rows;
    lf.links = o->links;
    lf.link_residual = o->link_residual;
    lf.mu_corr = c.ws + c.P.off_mucorr;
    lf.feas_residual = o->feas_residual;
    lf.status = o->status;
    lf.pool = c.ws + c.P.off_lfpool;
    if (plq::launch_link_feas(lf, c.s)) return cuda_fail("constrained link launch");
    ++nl;
  }
  g_launches += nl;
  return PLQ_OK;
}

plq::ReconArgs recon_args(const plq_problem_t* p, const plq_outputs_t* o, Ctx& c, int j0, int j1, double* part) {
  plq::ReconArgs a{};
  a.p = *p;
  a.Kx = o->K;
  a.Kz = c.Kz;
  a.k1 = c.k1;
  a.vf0 = o->vf0;
  a.links = o->links;
  a.k = o->k;
  a.x = o->x;
  a.u = o->u;
  a.lam = o->lam;
  a.mu_left = o->mu_left;
  a.lambda_right = o->lambda_right;
  a.gh = c.ws + c.P.off_gh;
  a.xend = c.ws + c.P.off_xend;
  a.part = part ? part : c.ws + c.P.off_part;
  a.seg_begin = j0;
  a.seg_end = j1;
  a.mu_corr = (o->feas && o->feas_rows && o->feas_residual) ? c.ws + c.P.off_mucorr : nullptr;
  a.feas_rows = o->feas_rows;
  return a;
}

int check_recon_out(const plq_outputs_t* o) {
  if (!o->K || !o->k || !o->x || !o->u || !o->lam || !o->links || !o->mu_left || !o->lambda_right || !o->vf0)
    return fail(PLQ_ERR_ARG, "null reconstruction output");
  return PLQ_OK;
}

int phase_recon(const plq_problem_t* p, const plq_outputs_t* o, Ctx& c, int j0, int j1, double* part) {
  int rc = check_recon_out(o);
  if (rc) return rc;
  if (j0 < 0 || j1 > p->J || j0 >= j1) return fail(PLQ_ERR_ARG, "bad segment range");
  const plq::ReconArgs ra = recon_args(p, o, c, j0, j1, part);
  if (use_small_recon(p) ? plq::launch_recon_small(ra, c.s) : plq::launch_recon(ra, c.s))
    return cuda_fail("recon launch");
  ++g_launches;
  return PLQ_OK;
}

int phase_boundary(const plq_problem_t* p, const plq_outputs_t* o, Ctx& c, int j0, int j1, double* part) {
  int rc = check_recon_out(o);
  if (rc) return rc;
  if (j0 < 0 || j1 > p->J || j0 >= j1) return fail(PLQ_ERR_ARG, "bad segment range");
  if (plq::launch_boundary(recon_args(p, o, c, j0, j1, part), nullptr, c.s)) return cuda_fail("boundary launch");
  ++g_launches;
  return PLQ_OK;
}

int phase_finalize(const plq_problem_t* p, const plq_outputs_t* o, Ctx& c, const double* part) {
  if (!o->objective || !o->kkt_inf || !o->link_mismatch || !o->mu_left || !o->lambda_right)
    return fail(PLQ_ERR_ARG, "null finalize output");
  if (plq::launch_finalize(*p, part ? part : c.ws + c.P.off_part, nullptr, o->mu_left, o->lambda_right, nullptr,
                           o->objective, o->kkt_inf, o->link_mismatch, nullptr, c.s))
    return cuda_fail("finalize launch");
  ++g_launches;
  return PLQ_OK;
}

}  // namespace

extern "C" {

int plq_abi_version(void) { return PLQ_ABI_VERSION; }

const char* plq_last_error(void) { return g_err; }

int plq_last_launch_count(void) { return g_launches; }

size_t plq_workspace_bytes(const plq_problem_t* problem) {
  if (check_problem(problem)) return 0;
  return make_plan(problem).total_doubles * sizeof(double);
}

int plq_solve_parallel(const plq_problem_t* problem, const plq_outputs_t* out, void* workspace,
                       size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Ctx c;
  int rc = setup(problem, out, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  const int J = problem->J;
  if ((rc = phase_sweep(problem, out, c, 0, J))) return rc;
  if ((rc = phase_link(problem, out, c))) return rc;
  if ((rc = phase_recon(problem, out, c, 0, J, nullptr))) return rc;
  if ((rc = phase_boundary(problem, out, c, 0, J, nullptr))) return rc;
  if ((rc = phase_finalize(problem, out, c, nullptr))) return rc;
  return PLQ_OK;
}

int plq_smooth(const plq_problem_t* problem, const plq_outputs_t* parent, const plq_smooth_outputs_t* out,
               void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Ctx c;
  int rc = setup(problem, parent, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  if (!out || !out->K || !out->k || !out->x || !out->u || !out->objective || !out->kkt_inf || !out->deviation ||
      !out->status)
    return fail(PLQ_ERR_ARG, "null smoothing output");
  if (!parent->K || !parent->k || !parent->x || !parent->u || !parent->lam || !parent->links || !parent->vf0)
    return fail(PLQ_ERR_ARG, "null parent solution field");
  const int J = problem->J;
  if (cudaMemsetAsync(out->status, 0, sizeof(int32_t) * problem->B * J, c.s) != cudaSuccess)
    return cuda_fail("status reset");
  if (J > 1) {
    plq::SweepArgs a{};
    a.p = *problem;
    a.Kx = out->K;
    a.Kz = c.ws + c.P.off_Kz;   // serial sweeps write Kz = 0: never into the parent's unfolded gains
    a.k1 = out->k;
    a.vf0 = nullptr;
    a.status = out->status;
    a.gscratch = c.ws + c.P.off_gs;
    a.task_ctr = reinterpret_cast<unsigned long long*>(c.ws + c.P.off_ctr);
    a.lay = c.P.lay;
    a.seg_begin = 0;
    a.seg_end = J - 1;
    a.smooth_vf0 = parent->vf0;
    a.smooth_links = parent->links;
    const int64_t tasks = problem->B * (int64_t)(J - 1);
    const int grid = (int)std::min<int64_t>(tasks, c.P.grid_max);
    rc = use_small_sweep(problem) ? plq::launch_sweep_small(a, c.s)
                                  : plq::launch_sweep(a, grid, c.P.threads, c.P.smem, c.s);
    if (rc) return cuda_fail("smoothing sweep launch");
    ++g_launches;
  }
  plq::SmoothArgs s{};
  s.p = *problem;
  s.K0 = parent->K;
  s.k0 = parent->k;
  s.x0 = parent->x;
  s.u0 = parent->u;
  s.lam0 = parent->lam;
  s.K = out->K;
  s.k = out->k;
  s.x = out->x;
  s.u = out->u;
  s.objective = out->objective;
  s.kkt = out->kkt_inf;
  s.deviation = out->deviation;
  s.maps = c.ws + c.P.off_smap;
  int nl = 0;
  if (plq::launch_smooth_rollout(s, c.s, &nl)) return cuda_fail("smoothing rollout launch");
  g_launches += nl;
  return PLQ_OK;
}

size_t plq_endpoint_workspace_bytes(const plq_problem_t* problem) {
  if (check_problem(problem) || problem->J != 1) return 0;
  return (make_plan(problem).total_doubles + up2(plq::endpoint_scratch_doubles(*problem)) +
          up2(plq::endpoint_eval_doubles(*problem))) * sizeof(double);
}

int plq_endpoint_affine(const plq_problem_t* problem, const plq_endpoint_outputs_t* out, void* workspace,
                        size_t workspace_bytes, void* stream) {
  g_launches = 0;
  if (check_problem(problem)) return PLQ_ERR_ARG;
  if (problem->J != 1) return fail(PLQ_ERR_ARG, "the two-point-boundary solve takes one segment (J = 1)");
  if (!out || !out->Kx || !out->Kz || !out->k1 || !out->value0 || !out->X || !out->S || !out->Lam || !out->E ||
      !out->status || !out->gram_status)
    return fail(PLQ_ERR_ARG, "null endpoint output");
  if (workspace_bytes < plq_endpoint_workspace_bytes(problem)) return fail(PLQ_ERR_WORKSPACE, "workspace too small");
  plq_outputs_t o{};
  o.K = out->Kx;
  o.Kz = out->Kz;
  o.k1 = out->k1;
  o.vf0 = out->value0;
  o.status = out->status;
  if ((out->feas != nullptr) != (out->feas_rows != nullptr)) return fail(PLQ_ERR_ARG, "feas and feas_rows go together");
  o.feas = out->feas;            // (B, J = 1, n, 2n+1): rows instead of PLQ_STATUS_DEGENERATE
  o.feas_rows = out->feas_rows;
  o.diag = out->diag;            // (B, J = 1, 2) / (B, J = 1)
  o.diag_rows = out->diag_rows;
  Ctx c;
  int rc = setup(problem, &o, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  if ((rc = phase_sweep(problem, &o, c, 0, 1, 1))) return rc;
  if (plq::launch_endpoint_maps_mult(*problem, *out, c.ws + c.P.total_doubles, c.s, &g_launches))
    return cuda_fail("endpoint maps / multiplier launch");
  return PLQ_OK;
}

int plq_endpoint_evaluate(const plq_problem_t* problem, const plq_endpoint_outputs_t* affine,
                          const plq_endpoint_point_t* point, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  if (check_problem(problem)) return PLQ_ERR_ARG;
  if (problem->J != 1) return fail(PLQ_ERR_ARG, "the two-point-boundary solve takes one segment (J = 1)");
  if (!affine || !affine->X || !affine->S || !affine->Lam || !affine->E) return fail(PLQ_ERR_ARG, "null maps");
  if (!point || !point->x_term || !point->x || !point->u || !point->lam || !point->mu || !point->objective ||
      !point->kkt_inf)
    return fail(PLQ_ERR_ARG, "null evaluation argument");
  if (!workspace || workspace_bytes < plq_endpoint_workspace_bytes(problem))
    return fail(PLQ_ERR_WORKSPACE, "workspace too small");
  const Plan P = make_plan(problem);
  double* ws = static_cast<double*>(workspace) + P.total_doubles + up2(plq::endpoint_scratch_doubles(*problem));
  if (plq::launch_endpoint_evaluate(*problem, *affine, *point, ws, static_cast<cudaStream_t>(stream), &g_launches))
    return cuda_fail("endpoint evaluation launch");
  return PLQ_OK;
}

int plq_sweep_segments(const plq_problem_t* problem, const plq_outputs_t* out, int32_t seg_begin, int32_t seg_end,
                       void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Ctx c;
  int rc = setup(problem, out, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  return phase_sweep(problem, out, c, seg_begin, seg_end);
}

int plq_link_solve(const plq_problem_t* problem, const plq_outputs_t* out, void* workspace, size_t workspace_bytes,
                   void* stream) {
  g_launches = 0;
  Ctx c;
  int rc = setup(problem, out, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  return phase_link(problem, out, c);
}

int plq_reconstruct_segments(const plq_problem_t* problem, const plq_outputs_t* out, int32_t seg_begin,
                             int32_t seg_end, double* partials, void* workspace, size_t workspace_bytes,
                             void* stream) {
  g_launches = 0;
  Ctx c;
  int rc = setup(problem, out, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  return phase_recon(problem, out, c, seg_begin, seg_end, partials);
}

int plq_boundary_segments(const plq_problem_t* problem, const plq_outputs_t* out, int32_t seg_begin,
                          int32_t seg_end, double* partials, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Ctx c;
  int rc = setup(problem, out, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  return phase_boundary(problem, out, c, seg_begin, seg_end, partials);
}

int plq_finalize(const plq_problem_t* problem, const plq_outputs_t* out, const double* partials, void* workspace,
                 size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Ctx c;
  int rc = setup(problem, out, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  return phase_finalize(problem, out, c, partials);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// device-side seeded generator

extern "C" int plq_generate_batch(const plq_problem_t* problem, const plq_recipe_t* recipe, void* stream) {
  g_launches = 0;
  const plq_problem_t* p = problem;
  if (!p || !recipe) return fail(PLQ_ERR_ARG, "null problem or recipe");
  if (p->B < 1 || p->T < 1 || p->n < 1 || p->m < 1 || p->n > 128 || p->m > 128)
    return fail(PLQ_ERR_ARG, "B, T >= 1 and 1 <= n, m <= 128");
  if (!p->Qxx || !p->Qux || !p->Quu || !p->qx1 || !p->qu1 || !p->Fx || !p->Fu || !p->f1 || !p->QxxT || !p->qx1T ||
      !p->x_init)
    return fail(PLQ_ERR_ARG, "null problem array");
  if (recipe->first_problem < 0 || recipe->first_problem + p->B > 0xffffffffLL)
    return fail(PLQ_ERR_ARG, "problem index out of range");
  if (plq::launch_generate(*p, recipe->a_scale, recipe->q_eps, recipe->r_eps, recipe->seed, recipe->first_problem,
                           static_cast<cudaStream_t>(stream)))
    return cuda_fail("generator launch");
  g_launches = 2;
  return PLQ_OK;
}

// ---------------------------------------------------------------------------
// horizon-sharded solve over an NCCL communicator

namespace {

// NCCL is bound at run time from the library the host process already uses
// (torch ships libnccl.so.2), so loading this library never needs NCCL.
struct NcclApi {
  void* h = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};
constexpr int kNcclInt32 = 2, kNcclFloat64 = 8;   // ncclDataType_t (nccl.h)

NcclApi& nccl_api() {
  static NcclApi a = [] {
    NcclApi x;
    const char* names[] = {getenv("PLQ_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm) continue;
      if ((x.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    }
    if (!x.h) return x;
    x.GroupStart = reinterpret_cast<int (*)()>(dlsym(x.h, "ncclGroupStart"));
    x.GroupEnd = reinterpret_cast<int (*)()>(dlsym(x.h, "ncclGroupEnd"));
    x.Broadcast = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
        dlsym(x.h, "ncclBroadcast"));
    x.AllGather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(
        dlsym(x.h, "ncclAllGather"));
    x.GetErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(x.h, "ncclGetErrorString"));
    x.ok = x.GroupStart && x.GroupEnd && x.Broadcast && x.AllGather;
    return x;
  }();
  return a;
}

inline void shard_range(int J, int nranks, int r, int* lo, int* hi) {
  const int base = J / nranks, extra = J % nranks;
  *lo = r * base + (r < extra ? r : extra);
  *hi = *lo + base + (r < extra ? 1 : 0);
}

// One in-place exchange of per-segment rows: buffer (B, Jrows, width) of
// `dtype`, rank r owning rows [lo_r + shift_lo, hi_r + shift_hi) clipped to
// [0, Jrows).  Equal contiguous shards of a single problem go as one in-place
// all-gather; everything else as grouped in-place broadcasts (one per owner
// and problem), which NCCL aggregates into one launch.
struct RowXfer {
  void* base;
  int64_t Jrows, width;   // rows per problem, elements per row
  int dtype, elem;        // NCCL type, bytes per element
  int shift;              // row index = segment index + shift (lambda_right rows: -1)
  int seg_lo_min, seg_hi_max;   // owned segments are clipped to [seg_lo_min, seg_hi_max)
};

int exchange_rows(const NcclApi& N, void* comm, int J, int nranks, int rank, int64_t B, const RowXfer* xs, int nx,
                  cudaStream_t s) {
  int rc = 0;
  const bool even = (J % nranks == 0) && B == 1;
  if ((rc = N.GroupStart())) return rc;
  for (int i = 0; i < nx && !rc; ++i) {
    const RowXfer& x = xs[i];
    const bool whole = even && x.shift == 0 && x.seg_lo_min == 0 && x.seg_hi_max == J;
    if (whole) {
      const size_t cnt = (size_t)(J / nranks) * x.width;
      char* b = static_cast<char*>(x.base);
      rc = N.AllGather(b + (size_t)rank * cnt * x.elem, b, cnt, x.dtype, comm, s);
      continue;
    }
    for (int r = 0; r < nranks && !rc; ++r) {
      int lo, hi;
      shard_range(J, nranks, r, &lo, &hi);
      lo = lo < x.seg_lo_min ? x.seg_lo_min : lo;
      hi = hi > x.seg_hi_max ? x.seg_hi_max : hi;
      if (hi <= lo) continue;
      for (int64_t b = 0; b < B && !rc; ++b) {
        char* ptr = static_cast<char*>(x.base) + ((size_t)b * x.Jrows + (lo + x.shift)) * x.width * x.elem;
        rc = N.Broadcast(ptr, ptr, (size_t)(hi - lo) * x.width, x.dtype, r, comm, s);
      }
    }
  }
  const int rc2 = N.GroupEnd();
  return rc ? rc : rc2;
}

}  // namespace

extern "C" int plq_solve_parallel_sharded(const plq_problem_t* problem, const plq_outputs_t* out, void* workspace,
                                          size_t workspace_bytes, void* nccl_comm, int32_t rank, int32_t nranks,
                                          void* stream) {
  g_launches = 0;
  Ctx c;
  int rc = setup(problem, out, workspace, workspace_bytes, stream, &c);
  if (rc) return rc;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PLQ_ERR_ARG, "bad rank / nranks");
  if (nranks > 1 && !nccl_comm) return fail(PLQ_ERR_ARG, "null communicator with nranks > 1");
  const bool feas = out->feas && out->feas_rows && out->feas_residual;
  if (!feas && (out->feas || out->feas_rows || out->feas_residual))
    return fail(PLQ_ERR_ARG, "feas, feas_rows and feas_residual go together");
  const NcclApi* N = nullptr;
  if (nccl_comm) {
    N = &nccl_api();
    if (!N->ok) return fail(PLQ_ERR_ARG, "NCCL (libnccl.so.2) could not be loaded; set PLQ_NCCL_LIB");
  }
  auto nccl_fail = [&](int e, const char* where) {
    snprintf(g_err, sizeof(g_err), "%s: NCCL error %d (%s)", where, e,
             N && N->GetErrorString ? N->GetErrorString(e) : "?");
    return PLQ_ERR_CUDA;
  };
  const int J = problem->J, n = problem->n;
  const int64_t B = problem->B;
  int j0, j1;
  shard_range(J, nranks, rank, &j0, &j1);
  double* part = c.ws + c.P.off_part;
  // 1. local sweeps; exchange of the segment-start value blocks, status and feasibility rows
  if (j1 > j0 && (rc = phase_sweep(problem, out, c, j0, j1))) return rc;
  if (N) {
    RowXfer xs[4] = {{out->vf0, J, (int64_t)3 * n * n + 2 * n, kNcclFloat64, 8, 0, 0, J},
                     {out->status, J, 1, kNcclInt32, 4, 0, 0, J},
                     {out->feas, J, (int64_t)n * (2 * n + 1), kNcclFloat64, 8, 0, 0, J},
                     {out->feas_rows, J, 1, kNcclInt32, 4, 0, 0, J}};
    const int e = exchange_rows(*N, nccl_comm, J, nranks, rank, B, xs, feas ? 4 : 2, c.s);
    if (e) return nccl_fail(e, "value-block exchange");
  }
  // 2. replicated coupling solve (bitwise identical on every rank)
  if ((rc = phase_link(problem, out, c))) return rc;
  // 3. local reconstruction; exchange of the multiplier rows at the links
  if (j1 > j0 && (rc = phase_recon(problem, out, c, j0, j1, part))) return rc;
  if (N && J > 1) {
    RowXfer xs[2] = {{out->mu_left, J - 1, n, kNcclFloat64, 8, 0, 0, J - 1},
                     {out->lambda_right, J - 1, n, kNcclFloat64, 8, -1, 1, J}};
    const int e = exchange_rows(*N, nccl_comm, J, nranks, rank, B, xs, 2, c.s);
    if (e) return nccl_fail(e, "multiplier-row exchange");
  }
  // 4. link-stage KKT rows; exchange of the per-segment partials; fixed-order reduction
  if (j1 > j0 && (rc = phase_boundary(problem, out, c, j0, j1, part))) return rc;
  if (N) {
    RowXfer xs[1] = {{part, J, 3, kNcclFloat64, 8, 0, 0, J}};
    const int e = exchange_rows(*N, nccl_comm, J, nranks, rank, B, xs, 1, c.s);
    if (e) return nccl_fail(e, "partials exchange");
  }
  return phase_finalize(problem, out, c, part);
}

extern "C" {

// ---------------------------------------------------------------------------
// host-buffer entry

namespace {

constexpr int NOUT_HOST = 19;   // plq_outputs_t fields copied back, in declaration order (diag / diag_rows are not)

void host_sizes(const plq_problem_t* p, size_t* in_sz, size_t* out_sz) {
  const size_t B = p->B, T = p->T, n = p->n, m = p->m, J = p->J;
  // order: split_times(int32), Qxx, Qux, Quu, qx1, qu1, Fx, Fu, f1, QxxT, qx1T, x_init (bytes)
  in_sz[0] = (J + 1) * sizeof(int32_t);
  in_sz[1] = B * T * n * n * 8;
  in_sz[2] = B * T * m * n * 8;
  in_sz[3] = B * T * m * m * 8;
  in_sz[4] = B * T * n * 8;
  in_sz[5] = B * T * m * 8;
  in_sz[6] = B * T * n * n * 8;
  in_sz[7] = B * T * n * m * 8;
  in_sz[8] = B * T * n * 8;
  in_sz[9] = B * n * n * 8;
  in_sz[10] = B * n * 8;
  in_sz[11] = B * n * 8;
  // order: K, k, x, u, lam, links, mu_left, lambda_right, vf0, Kz, k1, objective, kkt, mismatch, link_res, status
  out_sz[0] = B * T * m * n * 8;
  out_sz[1] = B * T * m * 8;
  out_sz[2] = B * (T + 1) * n * 8;
  out_sz[3] = B * T * m * 8;
  out_sz[4] = B * (T + 1) * n * 8;
  out_sz[5] = B * (J - 1) * n * 8;
  out_sz[6] = B * (J - 1) * n * 8;
  out_sz[7] = B * (J - 1) * n * 8;
  out_sz[8] = B * J * (3 * n * n + 2 * n) * 8;
  out_sz[9] = B * T * m * n * 8;
  out_sz[10] = B * T * m * 8;
  out_sz[11] = B * 8;
  out_sz[12] = B * 8;
  out_sz[13] = B * 8;
  out_sz[14] = B * 8;
  out_sz[15] = B * J * sizeof(int32_t);
  // degenerate partitions (parallel.py:320-384): feas, feas_rows, feas_residual
  out_sz[16] = B * J * n * (2 * n + 1) * 8;
  out_sz[17] = B * J * sizeof(int32_t);
  out_sz[18] = B * J * 8;
}

inline size_t up256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// Batches are processed in chunks of problems on three streams so the upload
// of chunk c+1, the solve of chunk c and the download of chunk c-1 overlap
// (PCIe / C2C is full duplex); a single problem is one chunk.
static void host_chunking(const plq_problem_t* hp, int* nchunks, int64_t* chunk_b, int* nstreams) {
  const int nc = hp->B >= 64 ? 8 : (hp->B >= 4 ? 4 : 1);
  *chunk_b = (hp->B + nc - 1) / nc;
  *nchunks = (int)((hp->B + *chunk_b - 1) / *chunk_b);
  *nstreams = *nchunks < 3 ? *nchunks : 3;
}

size_t plq_host_arena_bytes(const plq_problem_t* hp) {
  if (check_problem(hp)) return 0;
  size_t in_sz[12], out_sz[NOUT_HOST], total = 0;
  host_sizes(hp, in_sz, out_sz);
  for (size_t s : in_sz) total += up256(s);
  for (size_t s : out_sz) total += up256(s);
  int nc, ns;
  int64_t cb;
  host_chunking(hp, &nc, &cb, &ns);
  plq_problem_t c = *hp;
  c.B = cb;
  return total + (size_t)ns * up256(plq_workspace_bytes(&c));
}

int plq_solve_parallel_host(const plq_problem_t* hp, const plq_outputs_t* ho, void* arena, size_t arena_bytes,
                            void* stream) {
  int rc = check_problem(hp);
  if (rc) return rc;
  if (!ho || !arena) return fail(PLQ_ERR_ARG, "null outputs or arena");
  const size_t need = plq_host_arena_bytes(hp);
  if (arena_bytes < need) return fail(PLQ_ERR_WORKSPACE, "arena too small");
  // partition sanity on the host copy (parallel.py:434-440)
  for (int j = 0; j < hp->J; ++j)
    if (hp->split_times[j + 1] <= hp->split_times[j]) return fail(PLQ_ERR_ARG, "split times must be increasing");
  if (hp->split_times[0] != 0 || hp->split_times[hp->J] != hp->T)
    return fail(PLQ_ERR_ARG, "partition does not cover the horizon");
  cudaStream_t s0 = static_cast<cudaStream_t>(stream);
  size_t in_sz[12], out_sz[NOUT_HOST];
  host_sizes(hp, in_sz, out_sz);
  int nc, ns;
  int64_t cb;
  host_chunking(hp, &nc, &cb, &ns);
  char* cur = static_cast<char*>(arena);
  const void* hin[12] = {hp->split_times, hp->Qxx, hp->Qux, hp->Quu, hp->qx1, hp->qu1,
                         hp->Fx, hp->Fu, hp->f1, hp->QxxT, hp->qx1T, hp->x_init};
  char* din[12];
  for (int i = 0; i < 12; ++i) {
    din[i] = cur;
    cur += up256(in_sz[i]);
  }
  char* dout[NOUT_HOST];
  for (int i = 0; i < NOUT_HOST; ++i) {
    dout[i] = cur;
    cur += up256(out_sz[i]);
  }
  plq_problem_t cp = *hp;
  cp.B = cb;
  const size_t wsb = plq_workspace_bytes(&cp);
  char* wsp[3];
  for (int k = 0; k < ns; ++k) {
    wsp[k] = cur;
    cur += up256(wsb);
  }
  void* hout[NOUT_HOST] = {ho->K, ho->k, ho->x, ho->u, ho->lam, ho->links, ho->mu_left, ho->lambda_right,
                           ho->vf0, ho->Kz, ho->k1, ho->objective, ho->kkt_inf, ho->link_mismatch,
                           ho->link_residual, ho->status, ho->feas, ho->feas_rows, ho->feas_residual};
  cudaStream_t st[3] = {s0, nullptr, nullptr};
  cudaEvent_t ready = nullptr;
  for (int k = 1; k < ns; ++k)
    if (cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking) != cudaSuccess) return cuda_fail("stream create");
  if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess) return cuda_fail("event create");
  // the partition is shared by every chunk
  if (cudaMemcpyAsync(din[0], hin[0], in_sz[0], cudaMemcpyHostToDevice, s0) != cudaSuccess) rc = cuda_fail("H2D copy");
  cudaEventRecord(ready, s0);
  for (int k = 1; k < ns && !rc; ++k) cudaStreamWaitEvent(st[k], ready, 0);
  int launches = 0;
  for (int c = 0; c < nc && !rc; ++c) {
    cudaStream_t s = st[c % ns];
    const int64_t b0 = c * cb, bc = (b0 + cb <= hp->B) ? cb : hp->B - b0;
    // per-problem slice of every batched array: bytes per problem = total / B
    for (int i = 1; i < 12 && !rc; ++i) {
      const size_t per = in_sz[i] / (size_t)hp->B;
      if (cudaMemcpyAsync(din[i] + b0 * per, (const char*)hin[i] + b0 * per, bc * per, cudaMemcpyHostToDevice, s) !=
          cudaSuccess)
        rc = cuda_fail("H2D copy");
    }
    if (rc) break;
    plq_problem_t dp = *hp;
    dp.B = bc;
    dp.split_times = reinterpret_cast<const int32_t*>(din[0]);
    const double** fields[11] = {&dp.Qxx, &dp.Qux, &dp.Quu, &dp.qx1, &dp.qu1, &dp.Fx,
                                 &dp.Fu, &dp.f1, &dp.QxxT, &dp.qx1T, &dp.x_init};
    for (int i = 1; i < 12; ++i) *fields[i - 1] = reinterpret_cast<const double*>(din[i] + b0 * (in_sz[i] / hp->B));
    plq_outputs_t o{};   // feasibility buffers always on the device: degenerate partitions solved here too
    double** ofields[15] = {&o.K, &o.k, &o.x, &o.u, &o.lam, &o.links, &o.mu_left, &o.lambda_right,
                            &o.vf0, &o.Kz, &o.k1, &o.objective, &o.kkt_inf, &o.link_mismatch, &o.link_residual};
    for (int i = 0; i < 15; ++i) *ofields[i] = reinterpret_cast<double*>(dout[i] + b0 * (out_sz[i] / hp->B));
    o.status = reinterpret_cast<int32_t*>(dout[15] + b0 * (out_sz[15] / hp->B));
    o.feas = reinterpret_cast<double*>(dout[16] + b0 * (out_sz[16] / hp->B));
    o.feas_rows = reinterpret_cast<int32_t*>(dout[17] + b0 * (out_sz[17] / hp->B));
    o.feas_residual = reinterpret_cast<double*>(dout[18] + b0 * (out_sz[18] / hp->B));
    rc = plq_solve_parallel(&dp, &o, wsp[c % ns], wsb, s);
    launches += g_launches;
    if (rc) break;
    for (int i = 0; i < NOUT_HOST && !rc; ++i) {
      if (!hout[i]) continue;
      const size_t per = out_sz[i] / (size_t)hp->B;
      if (cudaMemcpyAsync((char*)hout[i] + b0 * per, dout[i] + b0 * per, bc * per, cudaMemcpyDeviceToHost, s) !=
          cudaSuccess)
        rc = cuda_fail("D2H copy");
    }
  }
  for (int k = 0; k < ns; ++k)
    if (cudaStreamSynchronize(st[k]) != cudaSuccess && !rc) rc = cuda_fail("stream sync");
  for (int k = 1; k < ns; ++k) cudaStreamDestroy(st[k]);
  cudaEventDestroy(ready);
  g_launches = launches;
  return rc;
}

}  // extern "C"

#ifdef PLQ_PHASE_PROFILE
namespace plq {
int sweep_small_phase_cycles(unsigned long long* out);
int sweep_phase_cycles_256(unsigned long long* out);
}
// Measurement builds only (-DPLQ_PHASE_PROFILE, libparlqr_b200_prof.so):
// per-CTA cycle counters of the specialized sweep's stage phases, 1024 x 16.
extern "C" int plq_debug_phase_cycles(unsigned long long* out) { return plq::sweep_small_phase_cycles(out); }
// the generic sweep's counters (256-thread instantiation)
extern "C" int plq_debug_phase_cycles_generic(unsigned long long* out) { return plq::sweep_phase_cycles_256(out); }
#endif
