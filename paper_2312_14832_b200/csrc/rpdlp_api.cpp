// C++ drop-in layer (include/rpdlp/*.hpp) over the C-ABI (include/pdhg.h).
//
// Problem-building storage (FromTriplets, VStack, StackK, Validate) stays on
// the host, with the reference's semantics (sparse_matrix.cpp:25-112,
// lp_problem.cpp:22-83). Solve, EstimateOpNorm, PrimalStep and DualStep run
// on the device through pdhg_*; C-ABI codes are rethrown as the reference's
// exception types.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>

#include "pdhg.h"
#include "rpdlp/solver.hpp"

namespace rpdlp {

// ------------------------------------------------------------ SparseMatrix
// Large inputs are assembled on the device (pdhg_csr_from_triplets: stable
// radix sort; duplicates summed in input order -- the same sums as here for
// up to two duplicates of an entry). Host path below that size, when the
// process sees no GPU (problem building is not the solve path), and for
// inputs with an entry duplicated three or more times (PDHG_ORDER_DEPENDENT:
// only the host's std::sort reproduces the reference's sum for those).
// Every other device failure (out of memory, a CUDA error) is thrown.
constexpr size_t kDeviceTriplets = size_t(1) << 20;

static bool DeviceAssemble(Index rows, Index cols, const std::vector<Triplet>& t, std::vector<Index>* rp,
                           std::vector<Index>* ci, std::vector<double>* val) {
  static_assert(sizeof(Triplet) == sizeof(pdhg_triplet), "Triplet layout");
  const char* da = std::getenv("PDHG_DEVICE_ASSEMBLY");  // "0": host only (A/B, tests)
  if (t.size() < kDeviceTriplets || (da && da[0] == '0') || pdhg_device_count() <= 0) return false;
  const char* dv = std::getenv("PDHG_DEVICE");
  rp->assign(rows + 1, 0);
  ci->resize(t.size());
  val->resize(t.size());
  int64_t nnz = 0;
  char err[512] = {0};
  const int rc = pdhg_csr_from_triplets(rows, cols, static_cast<int64_t>(t.size()),
                                        reinterpret_cast<const pdhg_triplet*>(t.data()), dv ? std::atoi(dv) : 0,
                                        rp->data(), ci->data(), val->data(), &nnz, err, sizeof(err));
  if (rc == PDHG_INVALID_ARGUMENT) throw std::out_of_range(err);
  if (rc == PDHG_ORDER_DEPENDENT) return false;
  if (rc != PDHG_OK) throw DeviceError(std::string("device triplet assembly: ") + err);
  ci->resize(nnz);
  val->resize(nnz);
  return true;
}

SparseMatrix SparseMatrix::FromTriplets(Index n_rows, Index n_cols, std::vector<Triplet> t) {
  if (n_rows < 0 || n_cols < 0) throw std::invalid_argument("negative matrix dimension");
  {
    SparseMatrix m;
    if (DeviceAssemble(n_rows, n_cols, t, &m.rp_, &m.ci_, &m.val_)) {
      m.rows_ = n_rows;
      m.cols_ = n_cols;
      m.BuildColumns();
      return m;
    }
  }
  for (const Triplet& e : t)
    if (e.row < 0 || e.row >= n_rows || e.col < 0 || e.col >= n_cols)
      throw std::out_of_range("triplet index out of range");
  std::sort(t.begin(), t.end(),
            [](const Triplet& a, const Triplet& b) { return std::tie(a.row, a.col) < std::tie(b.row, b.col); });
  SparseMatrix m;
  m.rows_ = n_rows;
  m.cols_ = n_cols;
  m.rp_.assign(n_rows + 1, 0);
  for (size_t i = 0; i < t.size();) {
    const Index r = t[i].row, c = t[i].col;
    double v = 0.0;
    for (; i < t.size() && t[i].row == r && t[i].col == c; ++i) v += t[i].value;
    if (v != 0.0) {
      m.ci_.push_back(c);
      m.val_.push_back(v);
      ++m.rp_[r + 1];
    }
  }
  for (Index r = 0; r < n_rows; ++r) m.rp_[r + 1] += m.rp_[r];
  m.BuildColumns();
  return m;
}

void SparseMatrix::BuildColumns() {
  cp_.assign(cols_ + 1, 0);
  ri_.assign(val_.size(), 0);
  cval_.assign(val_.size(), 0.0);
  for (Index j : ci_) ++cp_[j + 1];
  for (Index j = 0; j < cols_; ++j) cp_[j + 1] += cp_[j];
  std::vector<Index> fill(cp_.begin(), cp_.end() - 1);
  for (Index r = 0; r < rows_; ++r)
    for (Index k = rp_[r]; k < rp_[r + 1]; ++k) {
      const Index slot = fill[ci_[k]]++;
      ri_[slot] = r;
      cval_[slot] = val_[k];
    }
}

static void DeviceSpmv(const SparseMatrix& m, bool transpose, bool accumulate, double alpha,
                       std::span<const double> x, std::span<double> y) {
  const size_t nin = static_cast<size_t>(transpose ? m.rows() : m.cols());
  const size_t nout = static_cast<size_t>(transpose ? m.cols() : m.rows());
  if (x.size() != nin || y.size() != nout) throw std::invalid_argument("SpMV dimension mismatch");
  const pdhg_csr c{m.rows(), m.cols(), m.row_ptr().data(), m.col_idx().data(), m.csr_values().data()};
  char err[512] = {0};
  const int rc = pdhg_csr_spmv(&c, transpose ? 1 : 0, accumulate ? 1 : 0, alpha, x.data(), y.data(), err, sizeof(err));
  if (rc == PDHG_INVALID_ARGUMENT) throw std::invalid_argument(err);
  if (rc != PDHG_OK) throw DeviceError(err);
}

void SparseMatrix::Multiply(std::span<const double> x, std::span<double> y) const {
  DeviceSpmv(*this, false, false, 1.0, x, y);
}
void SparseMatrix::MultiplyTranspose(std::span<const double> x, std::span<double> y) const {
  DeviceSpmv(*this, true, false, 1.0, x, y);
}
void SparseMatrix::MultiplyAdd(double alpha, std::span<const double> x, std::span<double> y) const {
  DeviceSpmv(*this, false, true, alpha, x, y);
}
void SparseMatrix::MultiplyTransposeAdd(double alpha, std::span<const double> x, std::span<double> y) const {
  DeviceSpmv(*this, true, true, alpha, x, y);
}

static std::vector<double> DeviceNorms(const SparseMatrix& m, bool columns, bool power, double p) {
  std::vector<double> out(static_cast<size_t>(columns ? m.cols() : m.rows()), 0.0);
  const pdhg_csr c{m.rows(), m.cols(), m.row_ptr().data(), m.col_idx().data(), m.csr_values().data()};
  char err[512] = {0};
  const int rc = pdhg_csr_norms(&c, columns ? 1 : 0, power ? 1 : 0, p, out.data(), err, sizeof(err));
  if (rc == PDHG_INVALID_ARGUMENT) throw std::invalid_argument(err);
  if (rc != PDHG_OK) throw DeviceError(err);
  return out;
}

std::vector<double> SparseMatrix::RowInfNorms() const { return DeviceNorms(*this, false, false, 0.0); }
std::vector<double> SparseMatrix::ColInfNorms() const { return DeviceNorms(*this, true, false, 0.0); }
std::vector<double> SparseMatrix::RowPowerSums(double p) const { return DeviceNorms(*this, false, true, p); }
std::vector<double> SparseMatrix::ColPowerSums(double p) const { return DeviceNorms(*this, true, true, p); }

SparseMatrix SparseMatrix::Scaled(std::span<const double> row_scale, std::span<const double> col_scale) const {
  if (static_cast<Index>(row_scale.size()) != rows_ || static_cast<Index>(col_scale.size()) != cols_)
    throw std::invalid_argument("Scaled: scale length mismatch");
  SparseMatrix m = *this;
  const pdhg_csr c{rows_, cols_, rp_.data(), ci_.data(), val_.data()};
  char err[512] = {0};
  const int rc = pdhg_csr_scaled(&c, cp_.data(), ri_.data(), cval_.data(), row_scale.data(), col_scale.data(),
                                 m.val_.data(), m.cval_.data(), err, sizeof(err));
  if (rc == PDHG_INVALID_ARGUMENT) throw std::invalid_argument(err);
  if (rc != PDHG_OK) throw DeviceError(err);
  return m;
}

SparseMatrix SparseMatrix::VStack(const SparseMatrix& top, const SparseMatrix& bottom) {
  if (top.cols() != bottom.cols()) throw std::invalid_argument("VStack: column count mismatch");
  SparseMatrix m;
  m.rows_ = top.rows_ + bottom.rows_;
  m.cols_ = top.cols_;
  m.rp_ = top.rp_;
  for (size_t i = 1; i < bottom.rp_.size(); ++i) m.rp_.push_back(bottom.rp_[i] + top.nnz());
  m.ci_ = top.ci_;
  m.ci_.insert(m.ci_.end(), bottom.ci_.begin(), bottom.ci_.end());
  m.val_ = top.val_;
  m.val_.insert(m.val_.end(), bottom.val_.begin(), bottom.val_.end());
  m.BuildColumns();
  return m;
}

SparseMatrix SparseMatrix::RowSlice(Index begin, Index end) const {
  if (!(0 <= begin && begin <= end && end <= rows_)) throw std::out_of_range("RowSlice range");
  SparseMatrix m;
  m.rows_ = end - begin;
  m.cols_ = cols_;
  const Index base = rp_[begin];
  m.rp_.assign(1, 0);
  for (Index r = begin; r < end; ++r) m.rp_.push_back(rp_[r + 1] - base);
  m.ci_.assign(ci_.begin() + base, ci_.begin() + rp_[end]);
  m.val_.assign(val_.begin() + base, val_.begin() + rp_[end]);
  m.BuildColumns();
  return m;
}

std::vector<Triplet> SparseMatrix::ToTriplets() const {
  std::vector<Triplet> out;
  out.reserve(val_.size());
  for (Index r = 0; r < rows_; ++r)
    for (Index k = rp_[r]; k < rp_[r + 1]; ++k) out.push_back({r, ci_[k], val_[k]});
  return out;
}

// --------------------------------------------------------------- LpProblem
void LpProblem::Validate() const {
  const Index n = num_vars();
  if (a.cols() != n || g.cols() != n) throw std::invalid_argument("matrix column count does not match c");
  if (static_cast<Index>(b.size()) != a.rows()) throw std::invalid_argument("b length does not match A row count");
  if (static_cast<Index>(h.size()) != g.rows()) throw std::invalid_argument("h length does not match G row count");
  if (static_cast<Index>(l.size()) != n || static_cast<Index>(u.size()) != n)
    throw std::invalid_argument("bound vector length does not match c");
  auto nan_in = [](const std::vector<double>& v, const char* what) {
    for (double x : v)
      if (std::isnan(x)) throw std::invalid_argument(std::string("NaN in ") + what);
  };
  nan_in(c, "c");
  nan_in(b, "b");
  nan_in(h, "h");
  for (double x : c)
    if (std::isinf(x)) throw std::invalid_argument("infinite entry in c");
  for (Index i = 0; i < n; ++i) {
    if (std::isnan(l[i]) || std::isnan(u[i])) throw std::invalid_argument("NaN bound");
    if (l[i] > u[i]) throw std::invalid_argument("crossed bounds: l > u at index " + std::to_string(i));
  }
}

BoundClass ClassifyBound(double lower, double upper) {
  const bool lo = std::isfinite(lower), hi = std::isfinite(upper);
  if (lo && hi) return BoundClass::kBoxed;
  if (lo) return BoundClass::kLowerOnly;
  if (hi) return BoundClass::kUpperOnly;
  return BoundClass::kFree;
}

std::vector<BoundClass> ClassifyBounds(const LpProblem& p) {
  std::vector<BoundClass> out;
  out.reserve(p.l.size());
  for (size_t i = 0; i < p.l.size(); ++i) out.push_back(ClassifyBound(p.l[i], p.u[i]));
  return out;
}

std::pair<SparseMatrix, std::vector<double>> StackK(const LpProblem& p) {
  std::vector<double> q = p.b;
  q.insert(q.end(), p.h.begin(), p.h.end());
  return {SparseMatrix::VStack(p.a, p.g), std::move(q)};
}

// ------------------------------------------------------------- host helpers
bool CheckTermination(const ResidualReport& r, double eps) {
  return r.rel_primal <= eps && r.rel_dual <= eps && r.rel_gap <= eps;
}

double KktError(double p, double d, double g, double w) { return pdhg_kkt_error(p, d, g, w); }

namespace {

pdhg_params ToC(const SolverParams& s) {
  pdhg_params p;
  p.eps = s.eps;
  p.time_limit = s.time_limit;
  p.iter_limit = s.iter_limit;
  p.sufficient_decay = s.sufficient_decay;
  p.necessary_decay = s.necessary_decay;
  p.long_loop_frac = s.long_loop_frac;
  p.restart_enabled = s.restart_enabled;
  p.check_every = s.check_every;
  p.scaling_enabled = s.scaling.enabled;
  p.ruiz_iters = s.scaling.ruiz_iters;
  p.pc_alpha = s.scaling.pc_alpha;
  p.seed = s.seed;
  p.adaptive_step = s.adaptive_step;
  p.log_every = s.log_every;
  return p;
}

pdhg_csr View(const SparseMatrix& m) {
  return {m.rows(), m.cols(), m.row_ptr().data(), m.col_idx().data(), m.csr_values().data()};
}

pdhg_lp View(const LpProblem& p) {
  pdhg_lp v{};
  v.a = View(p.a);
  v.g = View(p.g);
  v.n = p.num_vars();
  v.c = p.c.data();
  v.b = p.b.data();
  v.h = p.h.data();
  v.l = p.l.data();
  v.u = p.u.data();
  v.objective_offset = p.objective_offset;
  v.negated_objective = p.negated_objective;
  return v;
}

ResidualReport FromC(const pdhg_report& r) {
  return {r.primal_res, r.dual_res, r.gap_abs, r.primal_obj, r.dual_obj, r.rel_primal, r.rel_dual, r.rel_gap};
}

[[noreturn]] void Rethrow(int code, const char* msg) {
  switch (code) {
    case PDHG_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case PDHG_NUMERICAL_FAILURE:
      throw NumericalFailure(msg);
    default:
      throw DeviceError(std::string("libpdhg_b200: ") + msg);
  }
}

int Device() {
  const char* d = std::getenv("PDHG_DEVICE");
  return d ? std::atoi(d) : 0;
}

struct ObserverCtx {
  const EvalObserver* fn;
  std::exception_ptr error;
};

int Trampoline(const pdhg_eval_info* c, void* user) {
  auto* ctx = static_cast<ObserverCtx*>(user);
  try {
    EvalInfo e;
    e.iteration = c->iteration;
    e.inner_iteration = c->inner_iteration;
    e.restarts = c->restarts;
    e.omega = c->omega;
    e.eta = c->eta;
    e.kkt_candidate = c->kkt_candidate;
    e.kkt_loop_start = c->kkt_loop_start;
    e.candidate_is_current = c->candidate_is_current != 0;
    e.restarted = c->restarted != 0;
    e.original_report = FromC(c->original_report);
    e.seconds = c->seconds;
    (*ctx->fn)(e);
    return 0;
  } catch (...) {
    ctx->error = std::current_exception();
    return 1;
  }
}

}  // namespace

void SolverParams::Validate() const {
  const pdhg_params p = ToC(*this);
  if (p.eps <= 0.0) throw std::invalid_argument("eps must be positive");
  if (!(0.0 < sufficient_decay && sufficient_decay < necessary_decay && necessary_decay < 1.0))
    throw std::invalid_argument("restart decay constants out of order");
  if (!(0.0 < long_loop_frac && long_loop_frac < 1.0)) throw std::invalid_argument("long_loop_frac must lie in (0, 1)");
  if (check_every < 1) throw std::invalid_argument("check_every must be >= 1");
  if (iter_limit < 0) throw std::invalid_argument("negative iter_limit");
}

std::string ToString(SolveStatus s) {
  switch (s) {
    case SolveStatus::kOptimal:
      return "Optimal";
    case SolveStatus::kIterLimit:
      return "IterLimit";
    case SolveStatus::kTimeLimit:
      return "TimeLimit";
  }
  return "Unknown";
}

bool ShouldRestart(const SolverParams& params, Index t, Index k, double cand, double start, double prev) {
  const pdhg_params p = ToC(params);
  return pdhg_should_restart(&p, t, k, cand, start, prev) != 0;
}

double UpdatePrimalWeight(double omega, double dx, double dy) { return pdhg_update_primal_weight(omega, dx, dy); }

void RunningAverage::Add(std::span<const double> x, std::span<const double> y) {
  const double w = weight_;
  for (size_t j = 0; j < x_.size(); ++j) x_[j] = (w * x_[j] + x[j]) / (w + 1.0);
  for (size_t i = 0; i < y_.size(); ++i) y_[i] = (w * y_[i] + y[i]) / (w + 1.0);
  weight_ = w + 1.0;
}

void RunningAverage::Reset() {
  std::fill(x_.begin(), x_.end(), 0.0);
  std::fill(y_.begin(), y_.end(), 0.0);
  weight_ = 0.0;
}

SolveResult Solve(const LpProblem& problem, const SolverParams& params, const EvalObserver& observer) {
  return Solve(problem, params, observer, DeviceOptions{});
}

SolveResult Solve(const LpProblem& problem, const SolverParams& params, const EvalObserver& observer,
                  const DeviceOptions& where) {
  if (where.shards < 1) throw std::invalid_argument("shards must be >= 1");
  problem.Validate();
  params.Validate();
  const pdhg_lp lp = View(problem);
  const pdhg_params prm = ToC(params);
  SolveResult r;
  r.x.resize(problem.num_vars());
  r.y.resize(problem.num_rows());
  r.lambda.resize(problem.num_vars());
  pdhg_result out{};
  out.x = r.x.data();
  out.y = r.y.data();
  out.lambda = r.lambda.data();
  ObserverCtx ctx{&observer, nullptr};
  char err[512] = {0};
  const int dev = where.device >= 0 ? where.device : Device();
  int code;
  if (where.shards == 1) {
    code = pdhg_solve_on(&lp, &prm, dev, observer ? Trampoline : nullptr, &ctx, &out, err, sizeof(err));
  } else {
    const pdhg_shard_spec spec{where.shards, 0, where.shards, nullptr};
    code = pdhg_solve_sharded(&lp, &prm, dev, &spec, observer ? Trampoline : nullptr, &ctx, &out, err, sizeof(err));
  }
  if (ctx.error) std::rethrow_exception(ctx.error);
  if (code != PDHG_OK) Rethrow(code, err);
  r.status = static_cast<SolveStatus>(out.status);
  r.report = FromC(out.report);
  r.iterations = out.iterations;
  r.restarts = out.restarts;
  r.solve_seconds = out.solve_seconds;
  r.scaling_seconds = out.scaling_seconds;
  return r;
}

double EstimateOpNorm(const SparseMatrix& k, int iters, std::uint64_t seed) {
  if (iters < 1) throw std::invalid_argument("iters must be >= 1");
  LpProblem p;
  p.a = SparseMatrix::FromTriplets(0, k.cols(), {});
  p.g = k;
  p.c.assign(k.cols(), 0.0);
  p.h.assign(k.rows(), 0.0);
  p.l.assign(k.cols(), 0.0);
  p.u.assign(k.cols(), 1.0);
  const pdhg_lp lp = View(p);
  pdhg_params prm;
  pdhg_params_default(&prm);
  prm.scaling_enabled = 0;
  pdhg_session* s = nullptr;
  char err[512] = {0};
  int code = pdhg_session_create(&lp, &prm, Device(), &s, err, sizeof(err));
  if (code != PDHG_OK) Rethrow(code, err);
  double out = 0.0;
  code = pdhg_session_opnorm(s, iters, seed, &out, err, sizeof(err));
  pdhg_session_destroy(s);
  if (code != PDHG_OK) Rethrow(code, err);
  return out;
}

std::vector<double> PrimalStep(const LpProblem& problem, std::span<const double> x, std::span<const double> y,
                               double eta, double omega) {
  const pdhg_lp lp = View(problem);
  std::vector<double> out(problem.num_vars());
  char err[512] = {0};
  const int code = pdhg_primal_step(&lp, x.data(), y.data(), eta, omega, out.data(), err, sizeof(err));
  if (code != PDHG_OK) Rethrow(code, err);
  return out;
}

std::vector<double> DualStep(const LpProblem& problem, std::span<const double> x_new, std::span<const double> x_old,
                             std::span<const double> y, double eta, double omega) {
  const pdhg_lp lp = View(problem);
  std::vector<double> out(problem.num_rows());
  char err[512] = {0};
  const int code =
      pdhg_dual_step(&lp, x_new.data(), x_old.data(), y.data(), eta, omega, out.data(), err, sizeof(err));
  if (code != PDHG_OK) Rethrow(code, err);
  return out;
}

}  // namespace rpdlp

// ------------------------------------------------------------- generators
#include "rpdlp/instance_gen.hpp"

namespace rpdlp {
namespace {

SparseMatrix FromCsr(const pdhg_csr& c) {
  std::vector<Triplet> t;
  const Index nz = c.rows ? c.row_ptr[c.rows] : 0;
  t.reserve(nz);
  for (Index r = 0; r < c.rows; ++r)
    for (Index k = c.row_ptr[r]; k < c.row_ptr[r + 1]; ++k) t.push_back({r, c.col_idx[k], c.values[k]});
  return SparseMatrix::FromTriplets(c.rows, c.cols, std::move(t));
}

LpProblem Take(pdhg_instance* inst, std::vector<double>* witness) {
  pdhg_lp v{};
  pdhg_instance_view(inst, &v);
  LpProblem p;
  p.name = pdhg_instance_name(inst);
  p.negated_objective = v.negated_objective != 0;
  p.a = FromCsr(v.a);
  p.g = FromCsr(v.g);
  p.c.assign(v.c, v.c + v.n);
  p.b.assign(v.b, v.b + v.a.rows);
  p.h.assign(v.h, v.h + v.g.rows);
  p.l.assign(v.l, v.l + v.n);
  p.u.assign(v.u, v.u + v.n);
  p.objective_offset = v.objective_offset;
  if (witness) {
    const double* w = pdhg_instance_witness(inst);
    if (w) witness->assign(w, w + v.n);
  }
  pdhg_instance_free(inst);
  return p;
}

}  // namespace

EdgeList GenPagerankGraph(const PagerankConfig& cfg) {
  EdgeList e(static_cast<size_t>(std::max<int64_t>(pdhg_pagerank_graph_edges(cfg.n_nodes, cfg.attachment), 0)));
  int64_t count = 0;
  char err[512] = {0};
  static_assert(sizeof(EdgeList::value_type) == 2 * sizeof(int64_t), "edge layout");
  if (pdhg_gen_pagerank_graph(cfg.n_nodes, cfg.damping, cfg.attachment, cfg.seed,
                              reinterpret_cast<int64_t*>(e.data()), static_cast<int64_t>(e.size()), &count, err,
                              sizeof(err)) != PDHG_OK)
    throw std::invalid_argument(err);
  e.resize(static_cast<size_t>(count));
  return e;
}

EdgeList ReadEdgeList(const std::string& path, Index* n_nodes) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  EdgeList edges;
  std::unordered_map<Index, Index> ids;  // raw id -> dense id, first appearance order
  auto dense = [&ids](Index raw) { return ids.emplace(raw, static_cast<Index>(ids.size())).first->second; };
  std::string line;
  while (std::getline(in, line)) {
    const size_t first = line.find_first_not_of(" \t\r");
    if (first == std::string::npos || line[first] == '#') continue;
    std::istringstream fields(line);
    Index src = 0, dst = 0;
    if (!(fields >> src >> dst)) throw std::runtime_error("malformed edge line: " + line);
    const Index a = dense(src);
    const Index b = dense(dst);
    edges.push_back({a, b});
  }
  if (n_nodes) *n_nodes = static_cast<Index>(ids.size());
  return edges;
}

LpProblem BuildPagerankLp(const EdgeList& edges, Index n_nodes, double damping) {
  pdhg_instance* inst = nullptr;
  char err[512] = {0};
  if (pdhg_build_pagerank_lp(reinterpret_cast<const int64_t*>(edges.data()), static_cast<int64_t>(edges.size()),
                             n_nodes, damping, &inst, err, sizeof(err)) != PDHG_OK)
    throw std::invalid_argument(err);
  LpProblem p = Take(inst, nullptr);
  p.name = "pagerank";
  p.Validate();
  return p;
}

LpProblem GenPagerank(const PagerankConfig& cfg) {
  pdhg_instance* inst = nullptr;
  char err[512] = {0};
  if (pdhg_gen_pagerank(cfg.n_nodes, cfg.damping, cfg.attachment, cfg.seed, &inst, err, sizeof(err)) != PDHG_OK)
    throw std::invalid_argument(err);
  LpProblem p = Take(inst, nullptr);
  p.name = "pagerank";
  return p;
}

LpProblem GenRandomLp(Index m, Index n, double density, std::uint64_t seed, std::vector<double>* witness) {
  pdhg_instance* inst = nullptr;
  char err[512] = {0};
  if (pdhg_gen_random_lp(m, n, density, seed, &inst, err, sizeof(err)) != PDHG_OK) throw std::invalid_argument(err);
  LpProblem p = Take(inst, witness);
  p.name = "rand_" + std::to_string(m) + "x" + std::to_string(n) + "_s" + std::to_string(seed);
  return p;
}

LpProblem GenTransport(Index sources, Index sinks, std::uint64_t seed) {
  pdhg_instance* inst = nullptr;
  char err[512] = {0};
  if (pdhg_gen_transport(sources, sinks, seed, &inst, err, sizeof(err)) != PDHG_OK) throw std::invalid_argument(err);
  return Take(inst, nullptr);
}

}  // namespace rpdlp

// ------------------------------------------------------------------- MPS
#include <fstream>
#include <iterator>
#include <sstream>

#include "rpdlp/mps.hpp"

namespace rpdlp {
namespace {

LpProblem FromMps(int code, pdhg_instance* inst, const char* err, int line) {
  if (code == PDHG_OK) return Take(inst, nullptr);
  std::string msg(err);
  if (code == PDHG_PARSE_ERROR) {
    const std::string prefix = "mps parse error at line " + std::to_string(line) + ": ";
    if (msg.compare(0, prefix.size(), prefix) == 0) msg = msg.substr(prefix.size());
    throw MpsParseError(line, msg);
  }
  if (code == PDHG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

}  // namespace

LpProblem ParseMpsString(const std::string& text, const MpsOptions& o) {
  pdhg_instance* inst = nullptr;
  char err[512] = {0};
  int line = 0;
  const int code = pdhg_mps_read_string(text.data(), text.size(), o.fixed_format, &inst, err, sizeof(err), &line);
  return FromMps(code, inst, err, line);
}

LpProblem ParseMps(std::istream& in, const MpsOptions& o) {
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return ParseMpsString(text, o);
}

LpProblem ParseMpsFile(const std::string& path, const MpsOptions& o) {
  pdhg_instance* inst = nullptr;
  char err[512] = {0};
  int line = 0;
  const int code = pdhg_mps_read_file(path.c_str(), o.fixed_format, &inst, err, sizeof(err), &line);
  return FromMps(code, inst, err, line);
}

void WriteMps(const LpProblem& problem, std::ostream& out) {
  const pdhg_lp v = View(problem);
  char* s = nullptr;
  size_t n = 0;
  char err[512] = {0};
  const int code = pdhg_mps_write_string(&v, problem.name.c_str(), &s, &n, err, sizeof(err));
  if (code == PDHG_INVALID_ARGUMENT) throw std::invalid_argument(err);
  if (code != PDHG_OK) throw std::runtime_error(err);
  out.write(s, static_cast<std::streamsize>(n));
  pdhg_free_string(s);
}

void WriteMpsFile(const LpProblem& problem, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  WriteMps(problem, out);
  out.flush();
  if (!out) throw std::runtime_error("write failed for " + path);
}

// SURVEY §8d configs 3 and 5 (not in the reference).
LpProblem GenMcf(Index nodes, Index arcs, Index commodities, std::uint64_t seed, std::vector<double>* witness) {
  pdhg_instance* inst = nullptr;
  char err[512] = {0};
  if (pdhg_gen_mcf(nodes, arcs, commodities, seed, &inst, err, sizeof(err)) != PDHG_OK)
    throw std::invalid_argument(err);
  return Take(inst, witness);
}

LpProblem GenStaircase(Index stages, Index rows_per_stage, Index cols_per_stage, Index nnz_per_row,
                       Index linking_per_row, Index eq_rows_per_stage, std::uint64_t seed,
                       std::vector<double>* witness) {
  pdhg_instance* inst = nullptr;
  char err[512] = {0};
  if (pdhg_gen_staircase(stages, rows_per_stage, cols_per_stage, nnz_per_row, linking_per_row, eq_rows_per_stage,
                         seed, 0, &inst, err, sizeof(err)) != PDHG_OK)
    throw std::invalid_argument(err);
  return Take(inst, witness);
}

}  // namespace rpdlp

// --------------------------------------------- scaling / residual utilities
#include "rpdlp/kkt.hpp"
#include "rpdlp/scaling.hpp"

namespace rpdlp {
namespace {

void Check(int code, const char* err) {
  if (code == PDHG_OK) return;
  if (code == PDHG_INVALID_ARGUMENT) throw std::invalid_argument(err);
  throw DeviceError(std::string("libpdhg_b200: ") + err);
}

ScalingInfo Scales(const SparseMatrix& k, int iters, double alpha, int stages) {
  ScalingInfo s{std::vector<double>(static_cast<size_t>(k.rows())), std::vector<double>(static_cast<size_t>(k.cols()))};
  const pdhg_csr c = View(k);
  char err[512] = {0};
  Check(pdhg_compute_scaling(&c, iters, alpha, stages, s.row_scale.data(), s.col_scale.data(), err, sizeof(err)), err);
  return s;
}

double Norm2(const std::vector<double>& v) {  // kkt.cpp:23-27 (sequential)
  double acc = 0.0;
  for (double e : v) acc += e * e;
  return std::sqrt(acc);
}

}  // namespace

ScalingInfo ScalingInfo::Identity(Index n_rows, Index n_cols) {
  return {std::vector<double>(static_cast<size_t>(n_rows), 1.0), std::vector<double>(static_cast<size_t>(n_cols), 1.0)};
}

ScalingInfo ScalingInfo::Composed(const ScalingInfo& other) const {
  ScalingInfo out = *this;
  for (size_t i = 0; i < out.row_scale.size(); ++i) out.row_scale[i] *= other.row_scale[i];
  for (size_t j = 0; j < out.col_scale.size(); ++j) out.col_scale[j] *= other.col_scale[j];
  return out;
}

void ScalingInfo::UnscaleIterate(std::span<double> x, std::span<double> y) const {
  for (size_t j = 0; j < x.size(); ++j) x[j] *= col_scale[j];
  for (size_t i = 0; i < y.size(); ++i) y[i] *= row_scale[i];
}

ScalingInfo RuizEquilibrate(const SparseMatrix& k, int iters) { return Scales(k, iters, 1.0, 1); }

ScalingInfo PockChambolleScale(const SparseMatrix& k, double alpha) {
  if (alpha < 0.0 || alpha > 2.0) throw std::invalid_argument("pock-chambolle alpha must lie in [0, 2]");
  return Scales(k, 0, alpha, 2);
}

ScalingInfo ComputeScaling(const SparseMatrix& k, const ScalingConfig& config) {
  if (!config.enabled) return ScalingInfo::Identity(k.rows(), k.cols());
  return Scales(k, config.ruiz_iters, config.pc_alpha, 3);
}

LpProblem ApplyScaling(const LpProblem& problem, const ScalingInfo& info) {
  const Index m1 = problem.num_eq_rows(), m2 = problem.num_ineq_rows();
  if (static_cast<Index>(info.row_scale.size()) != m1 + m2 ||
      static_cast<Index>(info.col_scale.size()) != problem.num_vars())
    throw std::invalid_argument("scaling dimensions do not match problem");
  auto scaled = [&](const SparseMatrix& m, Index r0) {
    std::vector<Triplet> t;
    for (Index r = 0; r < m.rows(); ++r)
      for (Index k = m.row_ptr()[r]; k < m.row_ptr()[r + 1]; ++k)
        t.push_back({r, m.col_idx()[k], (info.row_scale[r0 + r] * m.csr_values()[k]) * info.col_scale[m.col_idx()[k]]});
    return SparseMatrix::FromTriplets(m.rows(), m.cols(), std::move(t));
  };
  LpProblem out = problem;
  out.a = scaled(problem.a, 0);
  out.g = scaled(problem.g, m1);
  for (Index i = 0; i < m1; ++i) out.b[i] = problem.b[i] * info.row_scale[i];
  for (Index i = 0; i < m2; ++i) out.h[i] = problem.h[i] * info.row_scale[m1 + i];
  for (size_t j = 0; j < out.c.size(); ++j) {
    out.c[j] = problem.c[j] * info.col_scale[j];
    out.l[j] = problem.l[j] / info.col_scale[j];
    out.u[j] = problem.u[j] / info.col_scale[j];
  }
  return out;
}

std::vector<double> DeriveLambda(const LpProblem& problem, std::span<const double> y) {
  std::vector<double> out(static_cast<size_t>(problem.num_vars()));
  const pdhg_lp v = View(problem);
  char err[512] = {0};
  Check(pdhg_derive_lambda(&v, y.data(), out.data(), err, sizeof(err)), err);
  return out;
}

ResidualReport ComputeResiduals(const LpProblem& problem, const Iterate& z) {
  const pdhg_lp v = View(problem);
  pdhg_report r{};
  char err[512] = {0};
  Check(pdhg_residuals(&v, z.x.data(), z.y.data(), &r, err, sizeof(err)), err);
  return {r.primal_res, r.dual_res, r.gap_abs, r.primal_obj, r.dual_obj, r.rel_primal, r.rel_dual, r.rel_gap};
}

double KktOmega(const LpProblem& problem, const Iterate& z, double omega) {
  const ResidualReport r = ComputeResiduals(problem, z);
  return KktError(r.primal_res, r.dual_res, r.gap_abs, omega);
}

ResidualEvaluator::ResidualEvaluator(const LpProblem& problem) : problem_(problem) {
  std::vector<double> q(problem.b);
  q.insert(q.end(), problem.h.begin(), problem.h.end());
  q_norm_ = Norm2(q);
  c_norm_ = Norm2(problem.c);
}

ResidualReport ResidualEvaluator::Evaluate(std::span<const double> x, std::span<const double> y) const {
  return ComputeResiduals(problem_, Iterate{std::vector<double>(x.begin(), x.end()), std::vector<double>(y.begin(), y.end())});
}

double ResidualEvaluator::KktOmega(std::span<const double> x, std::span<const double> y, double omega) const {
  const ResidualReport r = Evaluate(x, y);
  return KktError(r.primal_res, r.dual_res, r.gap_abs, omega);
}

}  // namespace rpdlp

namespace rpdlp {

Iterate ChooseRestartCandidate(const LpProblem& problem, const Iterate& z_cur, const Iterate& z_avg, double omega) {
  const ResidualEvaluator ev(problem);  // both points on one device-resident problem
  const bool current = ev.KktOmega(z_cur.x, z_cur.y, omega) < ev.KktOmega(z_avg.x, z_avg.y, omega);
  return current ? z_cur : z_avg;
}

}  // namespace rpdlp

// C-ABI view of the drop-in's SparseMatrix::FromTriplets (device assembly
// for large inputs, the reference's std::sort on the host otherwise), so the
// Python mirror builds matrices with exactly the C++ drop-in's semantics.
extern "C" int pdhg_from_triplets(int64_t rows, int64_t cols, int64_t count, const pdhg_triplet* trips,
                                  int64_t* row_ptr, int64_t* col_idx, double* values, int64_t* nnz, char* err,
                                  size_t errlen) {
  auto put = [&](const char* m) {
    if (err && errlen) std::snprintf(err, errlen, "%s", m);
  };
  try {
    if (count < 0 || !row_ptr || !nnz || (count > 0 && (!trips || !col_idx || !values)))
      throw std::invalid_argument("null argument");
    std::vector<rpdlp::Triplet> t(static_cast<size_t>(count));
    if (count) std::memcpy(t.data(), trips, static_cast<size_t>(count) * sizeof(pdhg_triplet));
    const rpdlp::SparseMatrix m = rpdlp::SparseMatrix::FromTriplets(rows, cols, std::move(t));
    std::memcpy(row_ptr, m.row_ptr().data(), static_cast<size_t>(rows + 1) * sizeof(int64_t));
    const size_t k = m.col_idx().size();
    if (k) {
      std::memcpy(col_idx, m.col_idx().data(), k * sizeof(int64_t));
      std::memcpy(values, m.csr_values().data(), k * sizeof(double));
    }
    *nnz = static_cast<int64_t>(k);
    return PDHG_OK;
  } catch (const std::out_of_range& e) {
    put(e.what());
    return PDHG_INVALID_ARGUMENT;
  } catch (const std::invalid_argument& e) {
    put(e.what());
    return PDHG_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    put(e.what());
    return PDHG_CUDA_ERROR;
  }
}
