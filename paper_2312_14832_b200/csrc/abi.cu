// C-ABI entry points (include/pdhg.h). Exceptions never cross this boundary:
// every entry maps pdhg::Error / std::invalid_argument onto a return code and
// a message, which the C++ shim (include/rpdlp/) rethrows as the reference's
// exception types.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "assemble.cuh"
#include "host_logic.h"
#include "normal_rng.h"
#include "session.cuh"

struct pdhg_session {
  std::unique_ptr<pdhg::Session> impl;
};

namespace {

using pdhg::Error;

void put(char* err, size_t len, const std::string& m) {
  if (err && len) std::snprintf(err, len, "%s", m.c_str());
}

template <class F>
int Guard(char* err, size_t len, F&& f) {
  try {
    f();
    return PDHG_OK;
  } catch (const Error& e) {
    put(err, len, e.what());
    return e.code;
  } catch (const std::invalid_argument& e) {
    put(err, len, e.what());
    return PDHG_INVALID_ARGUMENT;
  } catch (const std::bad_alloc&) {
    put(err, len, "host allocation failed");
    return PDHG_CUDA_ERROR;
  } catch (const std::exception& e) {
    put(err, len, e.what());
    return PDHG_CUDA_ERROR;
  }
}

void Invalid(const std::string& m) { throw Error(PDHG_INVALID_ARGUMENT, m); }

// LpProblem::Validate (lp_problem.cpp:22-58), same checks and messages.
void ValidateLp(const pdhg_lp& lp) { pdhg::ValidateLpHost(lp); }

// SolverParams::Validate (solver.cpp:59-70).
void ValidateParams(const pdhg_params& p) {
  if (p.eps <= 0.0) Invalid("eps must be positive");
  if (!(0.0 < p.sufficient_decay && p.sufficient_decay < p.necessary_decay && p.necessary_decay < 1.0))
    Invalid("restart decay constants out of order");
  if (!(0.0 < p.long_loop_frac && p.long_loop_frac < 1.0)) Invalid("long_loop_frac must lie in (0, 1)");
  if (p.check_every < 1) Invalid("check_every must be >= 1");
  if (p.iter_limit < 0) Invalid("negative iter_limit");
}

// Device for the unit-level entry points ($PDHG_DEVICE, default 0), as the
// C++ shim chooses it for Solve.
int DeviceFromEnv() {
  const char* d = std::getenv("PDHG_DEVICE");
  return d ? std::atoi(d) : 0;
}

pdhg::ShardSpec Spec(const pdhg_shard_spec& s) {
  pdhg::ShardSpec r;
  r.world = s.world;
  r.rank = s.rank;
  r.local = s.local_shards;
  r.nccl_id = s.nccl_id;
  return r;
}

pdhg::Session& S(pdhg_session* s) {
  if (!s || !s->impl) Invalid("null session");
  return *s->impl;
}

}  // namespace

extern "C" {

void pdhg_params_default(pdhg_params* p) {
  p->eps = 1e-4;
  p->time_limit = 3600.0;
  p->iter_limit = INT64_MAX;
  p->sufficient_decay = 0.2;
  p->necessary_decay = 0.8;
  p->long_loop_frac = 0.36;
  p->restart_enabled = 1;
  p->check_every = 64;
  p->scaling_enabled = 1;
  p->ruiz_iters = 10;
  p->pc_alpha = 1.0;
  p->seed = 0;
  p->adaptive_step = 0;
  p->log_every = 0;
}

int pdhg_abi_version(void) { return PDHG_ABI_VERSION; }

const char* pdhg_build_info(void) {
  return "libpdhg_b200: sm_100a FP64 restarted PDHG (tile-segmented SpMV, fused step/check epilogues, CUDA graphs)";
}

int pdhg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int pdhg_session_create(const pdhg_lp* lp, const pdhg_params* prm, int device, pdhg_session** out, char* err,
                        size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!lp || !prm || !out) Invalid("null argument");
    ValidateLp(*lp);
    auto* s = new pdhg_session;
    try {
      s->impl = std::make_unique<pdhg::Session>(*lp, *prm, device);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int pdhg_session_create_sharded(const pdhg_lp* lp, const pdhg_params* prm, int device, const pdhg_shard_spec* spec,
                                pdhg_session** out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!lp || !prm || !out || !spec) Invalid("null argument");
    ValidateLp(*lp);
    auto* s = new pdhg_session;
    try {
      s->impl = std::make_unique<pdhg::Session>(*lp, *prm, device, Spec(*spec));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int pdhg_solve_sharded(const pdhg_lp* lp, const pdhg_params* prm, int device, const pdhg_shard_spec* spec,
                       pdhg_eval_cb cb, void* user, pdhg_result* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!lp || !prm || !out || !spec) Invalid("null argument");
    ValidateLp(*lp);
    ValidateParams(*prm);
    pdhg::Session sess(*lp, *prm, device, Spec(*spec));
    sess.Solve(*prm, cb, user, out);
  });
}

int pdhg_nccl_unique_id(void* out128, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!out128) Invalid("null argument");
    pdhg::nccl_unique_id(out128);
  });
}

int pdhg_loopback_id(void* out128, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!out128) Invalid("null argument");
    pdhg::loopback_id(out128);
  });
}

int pdhg_session_blocks(pdhg_session* s, int64_t* row_begin, int64_t* col_begin) {
  return Guard(nullptr, 0, [&] { S(s).Blocks(row_begin, col_begin); });
}

int pdhg_compute_scaling(const pdhg_csr* k, int ruiz_iters, double pc_alpha, int stages, double* row_scale,
                         double* col_scale, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!k || stages < 1 || stages > 3 || ruiz_iters < 0) Invalid("invalid scaling request");
    const int64_t n = k->cols, m = k->rows;
    std::vector<double> zn(static_cast<size_t>(n), 0.0), zm(static_cast<size_t>(m), 0.0);
    std::vector<int64_t> ap{0};
    pdhg_lp lp{};
    lp.a = {0, n, ap.data(), nullptr, nullptr};
    lp.g = *k;
    lp.n = n;
    lp.c = zn.data();
    lp.l = zn.data();
    lp.u = zn.data();
    lp.h = zm.data();
    ValidateLp(lp);
    pdhg_params p;
    pdhg_params_default(&p);
    p.scaling_enabled = 1;
    p.ruiz_iters = (stages & 1) ? ruiz_iters : 0;
    p.pc_alpha = pc_alpha;
    pdhg::Session sess(lp, p, DeviceFromEnv(), pdhg::ShardSpec{}, !(stages & 2));
    sess.Scaling(row_scale, col_scale);
  });
}

int pdhg_residuals(const pdhg_lp* lp, const double* x, const double* y, pdhg_report* out, char* err,
                   size_t errlen) {
  return Guard(err, errlen, [&] {
    // An empty iterate may come as a null pointer (std::vector{}.data()).
    if (!lp || !out || (!x && lp->n > 0) || (!y && lp->a.rows + lp->g.rows > 0)) Invalid("null argument");
    ValidateLp(*lp);
    pdhg_params p;
    pdhg_params_default(&p);
    p.scaling_enabled = 0;
    pdhg::Session sess(*lp, p, DeviceFromEnv());
    sess.Residuals(x, y, out);
  });
}

int pdhg_derive_lambda(const pdhg_lp* lp, const double* y, double* lambda, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!lp || (!lambda && lp->n > 0) || (!y && lp->a.rows + lp->g.rows > 0)) Invalid("null argument");
    ValidateLp(*lp);
    pdhg_params p;
    pdhg_params_default(&p);
    p.scaling_enabled = 0;
    pdhg::Session sess(*lp, p, DeviceFromEnv());
    sess.Lambda(y, lambda);
  });
}

int pdhg_session_ghost_counts(pdhg_session* s, int64_t* x_counts, int64_t* y_counts, int32_t* use) {
  return Guard(nullptr, 0, [&] { S(s).GhostCounts(x_counts, y_counts, use); });
}

int pdhg_partition_blocks(const int64_t* ptr, int64_t nseg, int parts, int64_t seg_weight, int64_t* begin) {
  if (!ptr || !begin || nseg < 0 || parts < 1 || seg_weight < 0) return PDHG_INVALID_ARGUMENT;
  pdhg::BalancedBlocks(ptr, nseg, parts, seg_weight, begin);
  return PDHG_OK;
}

void pdhg_session_destroy(pdhg_session* s) { delete s; }

int pdhg_normal_vector(uint64_t seed, int64_t n, int threads, double* out) {
  if (n < 0 || (n && !out)) return PDHG_INVALID_ARGUMENT;
  if (threads < 0) pdhg::NormalVectorSequential(seed, n, out);
  else pdhg::NormalVector(seed, n, out, threads);
  return PDHG_OK;
}

int pdhg_session_stats_get(pdhg_session* s, pdhg_session_stats* out) {
  return Guard(nullptr, 0, [&] { S(s).Stats(out); });
}

int pdhg_session_solve(pdhg_session* s, const pdhg_params* prm, pdhg_eval_cb cb, void* user, pdhg_result* out,
                       char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!prm || !out) Invalid("null argument");
    ValidateParams(*prm);
    if (!S(s).SameScaling(*prm))
      Invalid("solve params ask for a scaling (scaling.enabled, ruiz_iters, pc_alpha) other than the one the "
              "session was created with");
    S(s).Solve(*prm, cb, user, out);
  });
}

int pdhg_solve_on(const pdhg_lp* lp, const pdhg_params* prm, int device, pdhg_eval_cb cb, void* user,
                  pdhg_result* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!lp || !prm || !out) Invalid("null argument");
    const auto t0 = std::chrono::steady_clock::now();
    ValidateLp(*lp);
    ValidateParams(*prm);
    const auto t1 = std::chrono::steady_clock::now();
    double t2s = 0.0, t3s = 0.0;
    {
      pdhg::Session sess(*lp, *prm, device);
      const auto t2 = std::chrono::steady_clock::now();
      sess.Solve(*prm, cb, user, out);
      t2s = std::chrono::duration<double>(t2 - t1).count();
      t3s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();
    }
    if (std::getenv("PDHG_TRACE")) {
      const auto t4 = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[pdhg] pdhg_solve_on %.4fs: validate %.4fs | session %.4fs | solve %.4fs | teardown %.4fs\n",
                   std::chrono::duration<double>(t4 - t0).count(), std::chrono::duration<double>(t1 - t0).count(),
                   t2s, t3s, std::chrono::duration<double>(t4 - t1).count() - t2s - t3s);
    }
  });
}

int pdhg_solve(const pdhg_lp* lp, const pdhg_params* prm, pdhg_eval_cb cb, void* user, pdhg_result* out, char* err,
               size_t errlen) {
  return pdhg_solve_on(lp, prm, 0, cb, user, out, err, errlen);
}

int pdhg_session_scaling(pdhg_session* s, double* rs, double* cs, char* err, size_t errlen) {
  return Guard(err, errlen, [&] { S(s).Scaling(rs, cs); });
}

int pdhg_session_scaled(pdhg_session* s, double* kv, double* c, double* l, double* u, double* q, char* err,
                        size_t errlen) {
  return Guard(err, errlen, [&] { S(s).ScaledProblem(kv, c, l, u, q); });
}

int pdhg_session_spmv(pdhg_session* s, int transpose, const double* in, double* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] { S(s).Spmv(transpose, in, out); });
}

int pdhg_session_opnorm(pdhg_session* s, int iters, uint64_t seed, double* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (iters < 1) Invalid("iters must be >= 1");
    *out = S(s).OpNorm(iters, seed);
  });
}

int pdhg_session_time_kernels(pdhg_session* s, int iters, double* ms_primal, double* ms_dual, double* ms_iter,
                              char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (iters < 1) Invalid("iters must be >= 1");
    S(s).TimeKernels(iters, ms_primal, ms_dual, ms_iter);
  });
}

int pdhg_session_time_kernels_cold(pdhg_session* s, int iters, double* ms_primal, double* ms_dual,
                                   double* ms_iter, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (iters < 1) Invalid("iters must be >= 1");
    if (!ms_primal || !ms_dual || !ms_iter) Invalid("null argument");
    S(s).TimeKernelsCold(iters, ms_primal, ms_dual, ms_iter);
  });
}

int pdhg_session_run_block(pdhg_session* s, int iters, int profiler_range, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (iters < 1) Invalid("iters must be >= 1");
    S(s).RunBlock(iters, profiler_range != 0);
  });
}

int pdhg_session_time_check(pdhg_session* s, int iters, double* ms_device, double* ms_wall, char* err,
                            size_t errlen) {
  return Guard(err, errlen, [&] {
    if (iters < 1) Invalid("iters must be >= 1");
    S(s).TimeCheck(iters, ms_device, ms_wall);
  });
}

int pdhg_session_flush_l2(pdhg_session* s, char* err, size_t errlen) {
  return Guard(err, errlen, [&] { S(s).FlushL2(); });
}

int pdhg_session_last_solve(pdhg_session* s, double* device_ms, int64_t* kernel_launches) {
  return Guard(nullptr, 0, [&] {
    *device_ms = S(s).last_device_ms();
    *kernel_launches = S(s).last_launches();
  });
}

int pdhg_should_restart(const pdhg_params* p, int64_t t, int64_t k, double cand, double start, double prev) {
  return pdhg::ShouldRestart(*p, t, k, cand, start, prev) ? 1 : 0;
}

double pdhg_update_primal_weight(double omega, double dx, double dy) {
  return pdhg::UpdatePrimalWeight(omega, dx, dy);
}

double pdhg_kkt_error(double p, double d, double g, double w) { return pdhg::KktError(p, d, g, w); }

int pdhg_check_termination(const pdhg_report* r, double eps) { return pdhg::Terminated(*r, eps) ? 1 : 0; }

int pdhg_primal_step(const pdhg_lp* lp, const double* x, const double* y, double eta, double omega, double* out,
                     char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    ValidateLp(*lp);
    pdhg_params p;
    pdhg_params_default(&p);
    p.scaling_enabled = 0;
    pdhg::Session sess(*lp, p, 0);
    sess.UnitPrimal(x, y, eta, omega, out);
  });
}

}  // extern "C"

// A matrix as the inequality block of a free, zero-cost LP, unscaled: the
// session's K is the matrix itself (pdhg_csr_spmv / pdhg_csr_norms).
template <class F>
void WithMatrixSession(const pdhg_csr& m, F&& f) {
  static const int64_t kEmptyPtr[1] = {0};
  const int64_t n = m.cols;
  std::vector<double> zc(static_cast<size_t>(std::max<int64_t>(n, 1)), 0.0),
      lo(static_cast<size_t>(std::max<int64_t>(n, 1)), -INFINITY),
      hi(static_cast<size_t>(std::max<int64_t>(n, 1)), INFINITY), zh(static_cast<size_t>(std::max<int64_t>(m.rows, 1)), 0.0);
  pdhg_lp lp{};
  lp.a = pdhg_csr{0, n, kEmptyPtr, nullptr, nullptr};
  lp.g = m;
  lp.n = n;
  lp.c = zc.data();
  lp.l = lo.data();
  lp.u = hi.data();
  lp.h = zh.data();
  pdhg_params p;
  pdhg_params_default(&p);
  p.scaling_enabled = 0;
  pdhg::Session sess(lp, p, DeviceFromEnv());
  f(sess);
}

extern "C" {

int pdhg_csr_spmv(const pdhg_csr* m, int transpose, int accumulate, double alpha, const double* x, double* y,
                  char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!m || (m->rows < 0) || (m->cols < 0)) Invalid("bad matrix");
    const int64_t nin = transpose ? m->rows : m->cols, nout = transpose ? m->cols : m->rows;
    if ((nin && !x) || (nout && !y)) Invalid("null vector");
    if (nout == 0) return;
    std::vector<double> t(static_cast<size_t>(nout), 0.0);
    const int64_t nnz = m->rows ? m->row_ptr[m->rows] : 0;
    if (nnz > 0) WithMatrixSession(*m, [&](pdhg::Session& sess) { sess.Spmv(transpose, x, t.data()); });
    if (accumulate)
      for (int64_t i = 0; i < nout; ++i) y[i] += alpha * t[i];
    else
      std::copy(t.begin(), t.end(), y);
  });
}


int pdhg_csr_norms(const pdhg_csr* m, int columns, int power, double p, double* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!m || m->rows < 0 || m->cols < 0) Invalid("bad matrix");
    const int64_t nout = columns ? m->cols : m->rows;
    if (nout == 0) return;
    if (!out) Invalid("null vector");
    const int64_t nnz = m->rows ? m->row_ptr[m->rows] : 0;
    if (nnz == 0) {
      std::fill(out, out + nout, 0.0);
      return;
    }
    WithMatrixSession(*m, [&](pdhg::Session& s) { s.SegmentNorms(columns, power, p, out); });
  });
}

int pdhg_csr_scaled(const pdhg_csr* m, const int64_t* col_ptr, const int64_t* row_idx, const double* csc_values,
                    const double* row_scale, const double* col_scale, double* csr_out, double* csc_out, char* err,
                    size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!m || m->rows < 0 || m->cols < 0) Invalid("bad matrix");
    pdhg::ScaleEntries(*m, col_ptr, row_idx, csc_values, row_scale, col_scale, DeviceFromEnv(), csr_out, csc_out);
  });
}

int pdhg_dual_step(const pdhg_lp* lp, const double* xn, const double* xo, const double* y, double eta, double omega,
                   double* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    ValidateLp(*lp);
    pdhg_params p;
    pdhg_params_default(&p);
    p.scaling_enabled = 0;
    pdhg::Session sess(*lp, p, 0);
    sess.UnitDual(xn, xo, y, eta, omega, out);
  });
}

}  // extern "C"

int pdhg_csr_from_triplets(int64_t rows, int64_t cols, int64_t count, const pdhg_triplet* trips, int device,
                           int64_t* row_ptr, int64_t* col_idx, double* values, int64_t* nnz, char* err,
                           size_t errlen) {
  return Guard(err, errlen, [&] {
    if (!row_ptr || !nnz || (count > 0 && (!trips || !col_idx || !values))) Invalid("null argument");
    try {
      *nnz = pdhg::CsrFromTriplets(rows, cols, count, trips, device, row_ptr, col_idx, values);
    } catch (const std::out_of_range& e) {
      Invalid(e.what());
    }
  });
}
