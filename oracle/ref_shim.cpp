// ORACLE — TEST INFRASTRUCTURE ONLY (see rpdlp_oracle.cpp header).
//
// extern "C" shim over the UNMODIFIED reference rpdlp library, compiled by
// oracle/Makefile straight from /root/reference/proj/core/src into
// oracle/_ref/librpdlp_ref.so. It lets Python pin the restatement
// (liboracle.so) and the GPU product against the reference itself, and lets
// bench.py time the reference CPU solve (`--impl reference`,
// cpu_baseline.kind = "reference"). No reference source is copied here; only
// its public headers are included.

#include <cstdio>
#include <limits>
#include <random>
#include <cstring>
#include <sstream>
#include <string>
#include <stdexcept>
#include <vector>

#include "rpdlp/instance_gen.hpp"
#include "rpdlp/kkt.hpp"
#include "rpdlp/lp_problem.hpp"
#include "rpdlp/mps.hpp"
#include "rpdlp/scaling.hpp"
#include "rpdlp/solver.hpp"
#include "../include/pdhg.h"

using namespace rpdlp;

namespace {

SparseMatrix FromCsr(const pdhg_csr& v, Index n) {
  std::vector<Triplet> t;
  const Index nz = v.rows ? v.row_ptr[v.rows] : 0;
  t.reserve(static_cast<size_t>(nz));
  for (Index r = 0; r < v.rows; ++r)
    for (Index k = v.row_ptr[r]; k < v.row_ptr[r + 1]; ++k) t.push_back({r, v.col_idx[k], v.values[k]});
  return SparseMatrix::FromTriplets(v.rows, n, std::move(t));
}

LpProblem ToProblem(const pdhg_lp& v) {
  LpProblem p;
  p.a = FromCsr(v.a, v.n);
  p.g = FromCsr(v.g, v.n);
  p.c.assign(v.c, v.c + v.n);
  p.b.assign(v.b, v.b + v.a.rows);
  p.h.assign(v.h, v.h + v.g.rows);
  p.l.assign(v.l, v.l + v.n);
  p.u.assign(v.u, v.u + v.n);
  p.objective_offset = v.objective_offset;
  p.negated_objective = v.negated_objective != 0;
  return p;
}

SolverParams ToParams(const pdhg_params& q) {
  SolverParams p;
  p.eps = q.eps;
  p.time_limit = q.time_limit;
  p.iter_limit = q.iter_limit;
  p.sufficient_decay = q.sufficient_decay;
  p.necessary_decay = q.necessary_decay;
  p.long_loop_frac = q.long_loop_frac;
  p.restart_enabled = q.restart_enabled != 0;
  p.check_every = q.check_every;
  p.scaling.enabled = q.scaling_enabled != 0;
  p.scaling.ruiz_iters = q.ruiz_iters;
  p.scaling.pc_alpha = q.pc_alpha;
  p.seed = q.seed;
  p.adaptive_step = q.adaptive_step != 0;
  p.log_every = q.log_every;
  return p;
}

pdhg_report ToReport(const ResidualReport& r) {
  return {r.primal_res, r.dual_res, r.gap_abs, r.primal_obj, r.dual_obj, r.rel_primal, r.rel_dual, r.rel_gap};
}

template <class F>
int Guard(char* err, size_t len, F&& f) {
  auto put = [&](const char* m) {
    if (err && len) std::snprintf(err, len, "%s", m);
  };
  try {
    f();
    return PDHG_OK;
  } catch (const std::invalid_argument& e) {
    put(e.what());
    return PDHG_INVALID_ARGUMENT;
  } catch (const NumericalFailure& e) {
    put(e.what());
    return PDHG_NUMERICAL_FAILURE;
  } catch (const std::exception& e) {
    put(e.what());
    return PDHG_ABORTED;
  }
}

struct Abort {};

}  // namespace

struct ref_instance {
  LpProblem p;
  std::vector<double> witness;
};

extern "C" {

int ref_solve(const pdhg_lp* lp, const pdhg_params* prm, pdhg_eval_cb cb, void* user, pdhg_result* out, char* err,
              size_t errlen) {
  return Guard(err, errlen, [&] {
    LpProblem p = ToProblem(*lp);
    SolverParams sp = ToParams(*prm);
    EvalObserver obs = nullptr;
    if (cb) {
      obs = [&](const EvalInfo& e) {
        pdhg_eval_info c{};
        c.iteration = e.iteration;
        c.inner_iteration = e.inner_iteration;
        c.restarts = e.restarts;
        c.omega = e.omega;
        c.eta = e.eta;
        c.kkt_candidate = e.kkt_candidate;
        c.kkt_loop_start = e.kkt_loop_start;
        c.candidate_is_current = e.candidate_is_current;
        c.restarted = e.restarted;
        c.original_report = ToReport(e.original_report);
        c.seconds = e.seconds;
        if (cb(&c, user) != 0) throw std::runtime_error("aborted by observer");
      };
    }
    SolveResult r = Solve(p, sp, obs);
    out->status = static_cast<int32_t>(r.status);
    out->report = ToReport(r.report);
    out->iterations = r.iterations;
    out->restarts = r.restarts;
    out->solve_seconds = r.solve_seconds;
    out->scaling_seconds = r.scaling_seconds;
    if (out->x) std::memcpy(out->x, r.x.data(), r.x.size() * sizeof(double));
    if (out->y) std::memcpy(out->y, r.y.data(), r.y.size() * sizeof(double));
    if (out->lambda) std::memcpy(out->lambda, r.lambda.data(), r.lambda.size() * sizeof(double));
  });
}

int ref_scaling(const pdhg_lp* lp, const pdhg_params* prm, double* rs, double* cs, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    LpProblem p = ToProblem(*lp);
    auto [k, q] = StackK(p);
    ScalingConfig cfg{prm->scaling_enabled != 0, prm->ruiz_iters, prm->pc_alpha};
    ScalingInfo s = ComputeScaling(k, cfg);
    std::memcpy(rs, s.row_scale.data(), s.row_scale.size() * sizeof(double));
    std::memcpy(cs, s.col_scale.data(), s.col_scale.size() * sizeof(double));
  });
}

int ref_scaled(const pdhg_lp* lp, const pdhg_params* prm, double* kv, double* c, double* l, double* u, double* q,
               char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    LpProblem p = ToProblem(*lp);
    ScalingConfig cfg{prm->scaling_enabled != 0, prm->ruiz_iters, prm->pc_alpha};
    auto [k0, q0] = StackK(p);
    LpProblem s = cfg.enabled ? ApplyScaling(p, ComputeScaling(k0, cfg)) : p;
    auto [k, qq] = StackK(s);
    if (kv) std::memcpy(kv, k.csr_values().data(), k.csr_values().size() * sizeof(double));
    if (c) std::memcpy(c, s.c.data(), s.c.size() * sizeof(double));
    if (l) std::memcpy(l, s.l.data(), s.l.size() * sizeof(double));
    if (u) std::memcpy(u, s.u.data(), s.u.size() * sizeof(double));
    if (q) std::memcpy(q, qq.data(), qq.size() * sizeof(double));
  });
}

int ref_spmv(const pdhg_lp* lp, const pdhg_params* prm, int transpose, const double* in, double* out, char* err,
             size_t errlen) {
  return Guard(err, errlen, [&] {
    LpProblem p = ToProblem(*lp);
    ScalingConfig cfg{prm->scaling_enabled != 0, prm->ruiz_iters, prm->pc_alpha};
    auto [k0, q0] = StackK(p);
    LpProblem s = cfg.enabled ? ApplyScaling(p, ComputeScaling(k0, cfg)) : p;
    auto [k, qq] = StackK(s);
    if (transpose) {
      k.MultiplyTranspose(std::span<const double>(in, k.rows()), std::span<double>(out, k.cols()));
    } else {
      k.Multiply(std::span<const double>(in, k.cols()), std::span<double>(out, k.rows()));
    }
  });
}

int ref_opnorm(const pdhg_lp* lp, const pdhg_params* prm, int iters, uint64_t seed, double* out, char* err,
               size_t errlen) {
  return Guard(err, errlen, [&] {
    LpProblem p = ToProblem(*lp);
    ScalingConfig cfg{prm->scaling_enabled != 0, prm->ruiz_iters, prm->pc_alpha};
    auto [k0, q0] = StackK(p);
    LpProblem s = cfg.enabled ? ApplyScaling(p, ComputeScaling(k0, cfg)) : p;
    auto [k, qq] = StackK(s);
    *out = EstimateOpNorm(k, iters, seed);
  });
}

int ref_residuals(const pdhg_lp* lp, const double* x, const double* y, pdhg_report* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    LpProblem p = ToProblem(*lp);
    Iterate z{std::vector<double>(x, x + p.num_vars()), std::vector<double>(y, y + p.num_rows())};
    *out = ToReport(ComputeResiduals(p, z));
  });
}

int ref_primal_step(const pdhg_lp* lp, const double* x, const double* y, double eta, double omega, double* out,
                    char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    LpProblem p = ToProblem(*lp);
    auto r = PrimalStep(p, std::span<const double>(x, p.num_vars()), std::span<const double>(y, p.num_rows()), eta,
                        omega);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int ref_dual_step(const pdhg_lp* lp, const double* xn, const double* xo, const double* y, double eta, double omega,
                  double* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    LpProblem p = ToProblem(*lp);
    auto r = DualStep(p, std::span<const double>(xn, p.num_vars()), std::span<const double>(xo, p.num_vars()),
                      std::span<const double>(y, p.num_rows()), eta, omega);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

// Reference generators, for pinning the product's restated generators.
ref_instance* ref_gen_random_lp(int64_t m, int64_t n, double density, uint64_t seed) {
  auto* r = new ref_instance;
  r->p = GenRandomLp(m, n, density, seed, &r->witness);
  return r;
}
ref_instance* ref_gen_pagerank(int64_t n, double damping, int64_t att, uint64_t seed) {
  auto* r = new ref_instance;
  r->p = GenPagerank({n, damping, att, seed});
  return r;
}
// Config 2: transportation LP, built here through the
// reference's own SparseMatrix::FromTriplets so that bench.py's reference
// arm never loads the product library. Same draw order as the product's
// GenTransport (csrc/instance_gen.cpp Transport): demands d_j, supplies s_i
// (scaled to 1.2 sum d), then costs c_ij row-major; x_ij at column i*T + j;
// A = demand rows (= d_j), G = supply rows -sum_j x_ij >= -s_i, x >= 0.
// tests/test_oracle.py pins it bit-for-bit against the product generator.
ref_instance* ref_gen_transport(int64_t S, int64_t T, uint64_t seed) {
  auto* r = new ref_instance;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<double> d(T), s(S);
  double sd = 0.0, ss = 0.0;
  for (auto& v : d) sd += (v = 1.0 + unit(rng));
  for (auto& v : s) ss += (v = 1.0 + unit(rng));
  const double f = 1.2 * sd / ss;
  for (auto& v : s) v *= f;
  const Index n = S * T;
  LpProblem& p = r->p;
  p.c.resize(n);
  for (auto& v : p.c) v = unit(rng);
  std::vector<Triplet> ta, tg;
  ta.reserve(n);
  tg.reserve(n);
  for (Index i = 0; i < S; ++i)
    for (Index j = 0; j < T; ++j) {
      ta.push_back({j, i * T + j, 1.0});
      tg.push_back({i, i * T + j, -1.0});
    }
  p.a = SparseMatrix::FromTriplets(T, n, std::move(ta));
  p.g = SparseMatrix::FromTriplets(S, n, std::move(tg));
  p.b = d;
  p.h.resize(S);
  for (Index i = 0; i < S; ++i) p.h[i] = -s[i];
  p.l.assign(n, 0.0);
  p.u.assign(n, std::numeric_limits<double>::infinity());
  p.name = "transport";
  return r;
}

// SparseMatrix::FromTriplets (sparse_matrix.cpp:25-69) itself, for pinning
// the product's device and host assembly. Outputs caller-allocated like
// pdhg_csr_from_triplets; returns 1 with the message on an exception.
int ref_from_triplets(int64_t rows, int64_t cols, int64_t count, const pdhg_triplet* trips, int64_t* row_ptr,
                      int64_t* col_idx, double* values, int64_t* nnz, char* err, size_t errlen) {
  try {
    std::vector<Triplet> t(static_cast<size_t>(count));
    for (int64_t i = 0; i < count; ++i) t[i] = {trips[i].row, trips[i].col, trips[i].value};
    SparseMatrix m = SparseMatrix::FromTriplets(rows, cols, std::move(t));
    std::memcpy(row_ptr, m.row_ptr().data(), (rows + 1) * sizeof(int64_t));
    std::memcpy(col_idx, m.col_idx().data(), m.col_idx().size() * sizeof(int64_t));
    std::memcpy(values, m.csr_values().data(), m.csr_values().size() * sizeof(double));
    *nnz = static_cast<int64_t>(m.col_idx().size());
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// Solve a reference-owned instance in place (no CSR round trip): the
// reference arm's timed call.
int ref_solve_instance(const ref_instance* inst, const pdhg_params* prm, pdhg_result* out, char* err,
                       size_t errlen) {
  return Guard(err, errlen, [&] {
    SolveResult r = Solve(inst->p, ToParams(*prm));
    out->status = static_cast<int32_t>(r.status);
    out->report = ToReport(r.report);
    out->iterations = r.iterations;
    out->restarts = r.restarts;
    out->solve_seconds = r.solve_seconds;
    out->scaling_seconds = r.scaling_seconds;
  });
}

void ref_instance_view(const ref_instance* r, pdhg_lp* v) {
  const LpProblem& p = r->p;
  v->a = {p.a.rows(), p.a.cols(), p.a.row_ptr().data(), p.a.col_idx().data(), p.a.csr_values().data()};
  v->g = {p.g.rows(), p.g.cols(), p.g.row_ptr().data(), p.g.col_idx().data(), p.g.csr_values().data()};
  v->n = p.num_vars();
  v->c = p.c.data();
  v->b = p.b.data();
  v->h = p.h.data();
  v->l = p.l.data();
  v->u = p.u.data();
  v->objective_offset = p.objective_offset;
  v->negated_objective = p.negated_objective;
}
const double* ref_instance_witness(const ref_instance* r) { return r->witness.empty() ? nullptr : r->witness.data(); }
void ref_instance_free(ref_instance* r) { delete r; }
const char* ref_instance_name(const ref_instance* r) { return r->p.name.c_str(); }

// ParseMpsString / WriteMps (mps_reader.cpp, mps_writer.cpp) for pinning the
// product's MPS reader and writer. Returns 0, or 6 with *line set on
// MpsParseError, 1 on std::invalid_argument (Validate), 7 otherwise.
int ref_parse_mps(const char* text, size_t len, int fixed, ref_instance** out, char* err, size_t errlen, int* line) {
  *line = 0;
  try {
    auto* r = new ref_instance;
    try {
      MpsOptions o;
      o.fixed_format = fixed != 0;
      r->p = ParseMpsString(std::string(text, len), o);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
    return 0;
  } catch (const MpsParseError& e) {
    std::snprintf(err, errlen, "%s", e.what());
    *line = e.line();
    return 6;
  } catch (const std::invalid_argument& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    return 7;
  }
}

int ref_write_mps(const pdhg_lp* lp, const char* name, char* out, size_t cap, size_t* len) {
  try {
    LpProblem p = ToProblem(*lp);
    p.name = name ? name : "";
    std::ostringstream os;
    WriteMps(p, os);
    const std::string s = os.str();
    *len = s.size();
    if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

}  // extern "C"
