// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into or called by the
// product (paper_2312_14832_b200/). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg may load liboracle.so, and only as the checker.
//
// A serial CPU restatement of the reference restarted-PDHG solve path
// (rpdlp, /root/reference/proj/core). Each function cites the reference
// file:line it restates. Written in C++ (not C) so that the power-iteration
// start vector can use the same libstdc++ <random> engines as the reference
// (std::mt19937_64 + std::normal_distribution, solver.cpp:88-91); the pinned
// dependency is GCC 13.3 libstdc++ (same image on the CPU and GPU boxes).
//
// Parity pinning: tests/test_oracle.py checks this restatement against
// (a) the reference itself compiled from /root/reference into
//     oracle/_ref/librpdlp_ref.so (oracle/Makefile) when present, and
// (b) golden vectors produced by that reference build and committed under
//     tests/golden/ (tests/golden/make_golden.py), which travel to the GPU box.
//
// ABI: the pdhg_* structs of include/pdhg.h, entry points prefixed oracle_.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/pdhg.h"

namespace {

using I = int64_t;
using Vec = std::vector<double>;
const double kInfD = std::numeric_limits<double>::infinity();

struct NumFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Compressed matrix holding both layouts, as SparseMatrix does
// (sparse_matrix.hpp:36-102).
struct Mat {
  I rows = 0, cols = 0;
  std::vector<I> rp{0}, ci;  // CSR
  Vec rv;
  std::vector<I> cp{0}, ri;  // CSC
  Vec cv;

  // BuildCscFromCsr (sparse_matrix.cpp:71-88): stable column scatter in row
  // order, so row indices ascend inside each column.
  void BuildCsc() {
    cp.assign(cols + 1, 0);
    ri.assign(rv.size(), 0);
    cv.assign(rv.size(), 0.0);
    for (I j : ci) ++cp[j + 1];
    for (I j = 0; j < cols; ++j) cp[j + 1] += cp[j];
    std::vector<I> next(cp.begin(), cp.end() - 1);
    for (I r = 0; r < rows; ++r)
      for (I k = rp[r]; k < rp[r + 1]; ++k) {
        I d = next[ci[k]]++;
        ri[d] = r;
        cv[d] = rv[k];
      }
  }
  // Multiply (sparse_matrix.cpp:114-125): row-sequential sums.
  void Mul(const double* x, double* y) const {
    for (I r = 0; r < rows; ++r) {
      double acc = 0.0;
      for (I k = rp[r]; k < rp[r + 1]; ++k) acc += rv[k] * x[ci[k]];
      y[r] = acc;
    }
  }
  // MultiplyTranspose (sparse_matrix.cpp:127-138): column-sequential sums.
  void MulT(const double* x, double* y) const {
    for (I j = 0; j < cols; ++j) {
      double acc = 0.0;
      for (I k = cp[j]; k < cp[j + 1]; ++k) acc += cv[k] * x[ri[k]];
      y[j] = acc;
    }
  }
  // MultiplyTransposeAdd (sparse_matrix.cpp:153-164): y += alpha * (M^T x),
  // the column sum is completed first.
  void MulTAdd(double alpha, const double* x, double* y) const {
    for (I j = 0; j < cols; ++j) {
      double acc = 0.0;
      for (I k = cp[j]; k < cp[j + 1]; ++k) acc += cv[k] * x[ri[k]];
      y[j] += alpha * acc;
    }
  }
  // Scaled (sparse_matrix.cpp:206-222): (rs * v) * cs in both layouts.
  Mat Scaled(const double* rs, const double* cs) const {
    Mat m = *this;
    for (I r = 0; r < rows; ++r)
      for (I k = rp[r]; k < rp[r + 1]; ++k) m.rv[k] = rs[r] * rv[k] * cs[ci[k]];
    for (I j = 0; j < cols; ++j)
      for (I k = cp[j]; k < cp[j + 1]; ++k) m.cv[k] = rs[ri[k]] * cv[k] * cs[j];
    return m;
  }
  I nnz() const { return (I)rv.size(); }
};

Mat FromView(const pdhg_csr& v, I n) {
  Mat m;
  m.rows = v.rows;
  m.cols = n;
  m.rp.assign(v.row_ptr, v.row_ptr + v.rows + 1);
  I nz = m.rp.back();
  m.ci.assign(v.col_idx, v.col_idx + nz);
  m.rv.assign(v.values, v.values + nz);
  m.BuildCsc();
  return m;
}

// VStack (sparse_matrix.cpp:90-112).
Mat VStack(const Mat& top, const Mat& bot) {
  Mat m;
  m.rows = top.rows + bot.rows;
  m.cols = top.cols;
  m.rp = top.rp;
  for (size_t i = 1; i < bot.rp.size(); ++i) m.rp.push_back(bot.rp[i] + top.nnz());
  m.ci = top.ci;
  m.ci.insert(m.ci.end(), bot.ci.begin(), bot.ci.end());
  m.rv = top.rv;
  m.rv.insert(m.rv.end(), bot.rv.begin(), bot.rv.end());
  m.BuildCsc();
  return m;
}

struct Lp {
  Mat a, g;
  Vec c, b, h, l, u;
  double off = 0.0;
  I n() const { return (I)c.size(); }
  I m1() const { return a.rows; }
  I m2() const { return g.rows; }
};

Lp FromLp(const pdhg_lp& v) {
  Lp p;
  p.a = FromView(v.a, v.n);
  p.g = FromView(v.g, v.n);
  p.c.assign(v.c, v.c + v.n);
  p.b.assign(v.b, v.b + v.a.rows);
  p.h.assign(v.h, v.h + v.g.rows);
  p.l.assign(v.l, v.l + v.n);
  p.u.assign(v.u, v.u + v.n);
  p.off = v.objective_offset;
  return p;
}

// LpProblem::Validate (lp_problem.cpp:22-58).
void Validate(const pdhg_lp& v) {
  const I n = v.n;
  if (v.a.cols != n || v.g.cols != n) throw std::invalid_argument("matrix column count does not match c");
  for (I i = 0; i < n; ++i)
    if (std::isnan(v.c[i])) throw std::invalid_argument("NaN in c");
  for (I i = 0; i < v.a.rows; ++i)
    if (std::isnan(v.b[i])) throw std::invalid_argument("NaN in b");
  for (I i = 0; i < v.g.rows; ++i)
    if (std::isnan(v.h[i])) throw std::invalid_argument("NaN in h");
  for (I i = 0; i < n; ++i)
    if (std::isinf(v.c[i])) throw std::invalid_argument("infinite entry in c");
  for (I i = 0; i < n; ++i) {
    if (std::isnan(v.l[i]) || std::isnan(v.u[i])) throw std::invalid_argument("NaN bound");
    if (v.l[i] > v.u[i]) throw std::invalid_argument("crossed bounds: l > u at index " + std::to_string(i));
  }
}

// SolverParams::Validate (solver.cpp:59-70).
void ValidateParams(const pdhg_params& p) {
  if (p.eps <= 0.0) throw std::invalid_argument("eps must be positive");
  if (!(0.0 < p.sufficient_decay && p.sufficient_decay < p.necessary_decay && p.necessary_decay < 1.0))
    throw std::invalid_argument("restart decay constants out of order");
  if (!(0.0 < p.long_loop_frac && p.long_loop_frac < 1.0))
    throw std::invalid_argument("long_loop_frac must lie in (0, 1)");
  if (p.check_every < 1) throw std::invalid_argument("check_every must be >= 1");
  if (p.iter_limit < 0) throw std::invalid_argument("negative iter_limit");
}

double Norm2(const double* v, I n) {  // solver.cpp:27-31, kkt.cpp:23-27
  double acc = 0.0;
  for (I i = 0; i < n; ++i) acc += v[i] * v[i];
  return std::sqrt(acc);
}
double Clamp(double v, double lo, double hi) {  // solver.cpp:33-35
  return std::min(std::max(v, lo), hi);
}

// BoundClass (lp_problem.hpp:65, lp_problem.cpp:60-67): 0 free, 1 upper
// only, 2 lower only, 3 boxed. ProjectReducedCost (kkt.cpp:29-41).
int Cls(double lo, double hi) {
  bool a = std::isfinite(lo), b = std::isfinite(hi);
  return (!a && !b) ? 0 : (!a ? 1 : (!b ? 2 : 3));
}
double Proj(double v, int cls) {
  switch (cls) {
    case 0: return 0.0;
    case 1: return std::min(v, 0.0);
    case 2: return std::max(v, 0.0);
    default: return v;
  }
}

// ResidualEvaluator (kkt.cpp:45-125).
struct Eval {
  const Lp& p;
  std::vector<int> cls;
  double qn, cn;
  mutable Vec ax, gx, kty;
  explicit Eval(const Lp& pp) : p(pp), ax(pp.m1()), gx(pp.m2()), kty(pp.n()) {
    for (I j = 0; j < p.n(); ++j) cls.push_back(Cls(p.l[j], p.u[j]));
    cn = Norm2(p.c.data(), p.n());
    double s = 0.0;
    for (double v : p.b) s += v * v;
    for (double v : p.h) s += v * v;
    qn = std::sqrt(s);
  }
  pdhg_report Evaluate(const double* x, const double* y) const {
    const I m1 = p.m1(), m2 = p.m2(), n = p.n();
    pdhg_report r{};
    p.a.Mul(x, ax.data());
    p.g.Mul(x, gx.data());
    double ps = 0.0;
    for (I i = 0; i < m1; ++i) { double d = ax[i] - p.b[i]; ps += d * d; }
    for (I i = 0; i < m2; ++i) { double d = std::max(p.h[i] - gx[i], 0.0); ps += d * d; }
    r.primal_res = std::sqrt(ps);
    p.a.MulT(y, kty.data());
    p.g.MulTAdd(1.0, y + m1, kty.data());
    double ds = 0.0, bt = 0.0;
    for (I j = 0; j < n; ++j) {
      double red = p.c[j] - kty[j];
      double lam = Proj(red, cls[j]);
      double d = red - lam;
      ds += d * d;
      if (lam > 0.0) bt += p.l[j] * lam;
      else if (lam < 0.0) bt += p.u[j] * lam;
    }
    r.dual_res = std::sqrt(ds);
    double po = p.off;
    for (I j = 0; j < n; ++j) po += p.c[j] * x[j];
    double dob = p.off + bt;
    for (I i = 0; i < m1; ++i) dob += p.b[i] * y[i];
    for (I i = 0; i < m2; ++i) dob += p.h[i] * y[m1 + i];
    r.primal_obj = po;
    r.dual_obj = dob;
    r.gap_abs = std::abs(dob - po);
    r.rel_primal = r.primal_res / (1.0 + qn);
    r.rel_dual = r.dual_res / (1.0 + cn);
    r.rel_gap = r.gap_abs / (1.0 + std::abs(dob) + std::abs(po));
    return r;
  }
};

double Kkt(double p, double d, double g, double w) {  // kkt.cpp:153-157
  return std::sqrt(w * w * p * p + d * d / (w * w) + g * g);
}
bool Terminate(const pdhg_report& r, double eps) {  // kkt.cpp:147-151
  return r.rel_primal <= eps && r.rel_dual <= eps && r.rel_gap <= eps;
}

// Ruiz (scaling.cpp:49-68), PC (scaling.cpp:70-84), ComputeScaling (:86-91).
void InfNorms(const Mat& k, Vec& rn, Vec& cn) {  // sparse_matrix.cpp:166-184
  rn.assign(k.rows, 0.0);
  cn.assign(k.cols, 0.0);
  for (I r = 0; r < k.rows; ++r)
    for (I q = k.rp[r]; q < k.rp[r + 1]; ++q) rn[r] = std::max(rn[r], std::abs(k.rv[q]));
  for (I j = 0; j < k.cols; ++j)
    for (I q = k.cp[j]; q < k.cp[j + 1]; ++q) cn[j] = std::max(cn[j], std::abs(k.cv[q]));
}
void ComputeScaling(const Mat& k, const pdhg_params& prm, Vec& rs, Vec& cs) {
  rs.assign(k.rows, 1.0);
  cs.assign(k.cols, 1.0);
  if (!prm.scaling_enabled) return;
  Mat w = k;
  Vec rn, cn;
  for (int s = 0; s < prm.ruiz_iters; ++s) {
    InfNorms(w, rn, cn);
    Vec dr(k.rows, 1.0), dc(k.cols, 1.0);
    for (I i = 0; i < k.rows; ++i) if (rn[i] > 0.0) dr[i] = 1.0 / std::sqrt(rn[i]);
    for (I j = 0; j < k.cols; ++j) if (cn[j] > 0.0) dc[j] = 1.0 / std::sqrt(cn[j]);
    w = w.Scaled(dr.data(), dc.data());
    for (I i = 0; i < k.rows; ++i) rs[i] *= dr[i];
    for (I j = 0; j < k.cols; ++j) cs[j] *= dc[j];
  }
  const double alpha = prm.pc_alpha;
  if (alpha < 0.0 || alpha > 2.0) throw std::invalid_argument("pock-chambolle alpha must lie in [0, 2]");
  Mat sc = k.Scaled(rs.data(), cs.data());
  // RowPowerSums / ColPowerSums (sparse_matrix.cpp:186-204).
  Vec rsum(k.rows, 0.0), csum(k.cols, 0.0);
  for (I r = 0; r < k.rows; ++r)
    for (I q = sc.rp[r]; q < sc.rp[r + 1]; ++q) rsum[r] += std::pow(std::abs(sc.rv[q]), 2.0 - alpha);
  for (I j = 0; j < k.cols; ++j)
    for (I q = sc.cp[j]; q < sc.cp[j + 1]; ++q) csum[j] += std::pow(std::abs(sc.cv[q]), alpha);
  for (I i = 0; i < k.rows; ++i) if (rsum[i] > 0.0) rs[i] *= 1.0 / std::sqrt(rsum[i]);
  for (I j = 0; j < k.cols; ++j) if (csum[j] > 0.0) cs[j] *= 1.0 / std::sqrt(csum[j]);
}

// ApplyScaling (scaling.cpp:93-116).
Lp ApplyScaling(const Lp& p, const Vec& rs, const Vec& cs) {
  Lp o = p;
  const I m1 = p.m1();
  o.a = p.a.Scaled(rs.data(), cs.data());
  o.g = p.g.Scaled(rs.data() + m1, cs.data());
  for (I i = 0; i < m1; ++i) o.b[i] = p.b[i] * rs[i];
  for (I i = 0; i < p.m2(); ++i) o.h[i] = p.h[i] * rs[m1 + i];
  for (I j = 0; j < p.n(); ++j) {
    o.c[j] = p.c[j] * cs[j];
    o.l[j] = p.l[j] / cs[j];
    o.u[j] = p.u[j] / cs[j];
  }
  return o;
}

// EstimateOpNorm (solver.cpp:84-110).
double OpNorm(const Mat& k, int iters, uint64_t seed) {
  if (k.nnz() == 0) return 0.0;
  const I n = k.cols;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  Vec v(n), kv(k.rows);
  for (double& e : v) e = gauss(rng);
  double vn = Norm2(v.data(), n);
  if (vn == 0.0) { v[0] = 1.0; vn = 1.0; }
  for (double& e : v) e /= vn;
  for (int it = 0; it < iters; ++it) {
    k.Mul(v.data(), kv.data());
    k.MulT(kv.data(), v.data());
    double nr = Norm2(v.data(), n);
    if (nr == 0.0) return 0.0;
    for (double& e : v) e /= nr;
  }
  k.Mul(v.data(), kv.data());
  return Norm2(kv.data(), k.rows);
}

// SolveLoop (solver.cpp:203-517), restated.
struct Loop {
  const Lp& orig;
  const Lp& sc;
  const Vec& rs;
  const Vec& cs;
  const pdhg_params& prm;
  pdhg_eval_cb cb;
  void* user;
  I m1, m, n;
  Mat k;
  Vec q;
  Eval se, oe;
  double eta = 1.0, omega = 1.0;
  Vec x, y, xs, ys, ax, ay, kty, kxc, kxn, xn, yn, ux, uy, bx, by;
  double avg_w = 0.0;
  double kkt_start = 0.0, kkt_prev = kInfD;
  I inner = 0, iters = 0, restarts = 0;
  pdhg_report best_rep{}, last_rep{};
  double best_k1 = 0.0;
  bool have_best = false;
  int status = PDHG_ITER_LIMIT;
  I last_log = -1;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();

  Loop(const Lp& o, const Lp& s, const Vec& r, const Vec& c, const pdhg_params& p, pdhg_eval_cb f, void* u)
      : orig(o), sc(s), rs(r), cs(c), prm(p), cb(f), user(u), m1(s.m1()), m(s.m1() + s.m2()), n(s.n()),
        se(s), oe(o) {
    k = VStack(sc.a, sc.g);  // StackK (lp_problem.cpp:78-83)
    q = sc.b;
    q.insert(q.end(), sc.h.begin(), sc.h.end());
    ax.assign(n, 0.0); ay.assign(m, 0.0); kty.resize(n); kxc.resize(m); kxn.resize(m);
    xn.resize(n); yn.resize(m); ux.resize(n); uy.resize(m);
  }
  double Secs() const {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  void Kx(const Vec& v, Vec& out) {  // ComputeKx (solver.cpp:270-273)
    sc.a.Mul(v.data(), out.data());
    sc.g.Mul(v.data(), out.data() + m1);
  }
  void StartAt() {  // StartLoopAt (solver.cpp:275-281)
    xs = x; ys = y;
    pdhg_report r = se.Evaluate(x.data(), y.data());
    kkt_start = Kkt(r.primal_res, r.dual_res, r.gap_abs, omega);
    kkt_prev = kInfD;
    std::fill(ax.begin(), ax.end(), 0.0);
    std::fill(ay.begin(), ay.end(), 0.0);
    avg_w = 0.0;
    inner = 0;
  }
  void Step() {  // solver.cpp:284-306
    k.MulT(y.data(), kty.data());
    const double ps = eta / omega;
    for (I j = 0; j < n; ++j) xn[j] = Clamp(x[j] - ps * (sc.c[j] - kty[j]), sc.l[j], sc.u[j]);
    k.Mul(xn.data(), kxn.data());
    const double ds = eta * omega;
    for (I i = 0; i < m; ++i) {
      double v = y[i] + ds * (q[i] - (2.0 * kxn[i] - kxc[i]));
      yn[i] = i < m1 ? v : std::max(v, 0.0);
    }
    if (prm.adaptive_step) Adapt();
    std::swap(x, xn);
    std::swap(y, yn);
    std::swap(kxc, kxn);
    const double w = avg_w;  // RunningAverage::Add (solver.cpp:156-162)
    for (I j = 0; j < n; ++j) ax[j] = (w * ax[j] + x[j]) / (w + 1.0);
    for (I i = 0; i < m; ++i) ay[i] = (w * ay[i] + y[i]) / (w + 1.0);
    avg_w = w + 1.0;
    ++inner;
    ++iters;
  }
  void Adapt() {  // AdaptStepSize (solver.cpp:310-328)
    double dx = 0.0, dy = 0.0, it = 0.0;
    for (I j = 0; j < n; ++j) { double d = xn[j] - x[j]; dx += d * d; }
    for (I i = 0; i < m; ++i) {
      double d = yn[i] - y[i];
      dy += d * d;
      it += d * (kxn[i] - kxc[i]);
    }
    it = std::abs(it);
    if (it <= 0.0) return;
    double lim = (omega * dx + dy / omega) / (2.0 * it);
    double kk = (double)(iters + 1);
    eta = std::min(lim * (1.0 - std::pow(kk, -0.3)), eta * (1.0 + std::pow(kk, -0.6)));
  }
  bool EvalOrig(const Vec& zx, const Vec& zy, pdhg_report* r) {  // solver.cpp:330-339
    for (I j = 0; j < n; ++j) ux[j] = zx[j] * cs[j];
    for (I i = 0; i < m; ++i) uy[i] = zy[i] * rs[i];
    *r = oe.Evaluate(ux.data(), uy.data());
    return Terminate(*r, prm.eps);
  }
  void RecordBest(const pdhg_report& r) {  // solver.cpp:341-351
    double k1 = Kkt(r.primal_res, r.dual_res, r.gap_abs, 1.0);
    if (!have_best || k1 < best_k1) {
      have_best = true;
      best_k1 = k1;
      bx = ux;
      by = uy;
      best_rep = r;
    }
  }
  bool EvalAndMaybeFinish(const Vec& cx, const Vec& cy, const Vec* vx, const Vec* vy) {  // :355-387
    pdhg_report r;
    if (EvalOrig(cx, cy, &r)) {
      status = PDHG_OPTIMAL; bx = ux; by = uy; best_rep = r; have_best = true; last_rep = r;
      return true;
    }
    RecordBest(r);
    last_rep = r;
    if (vx) {
      pdhg_report a;
      if (EvalOrig(*vx, *vy, &a)) {
        status = PDHG_OPTIMAL; bx = ux; by = uy; best_rep = a; have_best = true; last_rep = a;
        return true;
      }
      RecordBest(a);
      if (Kkt(a.primal_res, a.dual_res, a.gap_abs, 1.0) < Kkt(r.primal_res, r.dual_res, r.gap_abs, 1.0))
        last_rep = a;
    }
    return false;
  }
  static bool ShouldRestart(const pdhg_params& p, I t, I kk, double cand, double start, double prev) {
    if (cand <= p.sufficient_decay * start) return true;  // solver.cpp:178-189
    if (cand <= p.necessary_decay * start && cand > prev) return true;
    return (double)t >= p.long_loop_frac * (double)kk;
  }
  static double UpdateOmega(double w, double dx, double dy) {  // solver.cpp:191-196
    if (dx <= 1e-10 || dy <= 1e-10) return w;
    return std::exp(0.5 * std::log(dy / dx) + 0.5 * std::log(w));
  }
  bool Check() {  // solver.cpp:390-428
    for (double v : x) if (!std::isfinite(v)) throw NumFail("non-finite iterate at iteration " + std::to_string(iters));
    for (double v : y) if (!std::isfinite(v)) throw NumFail("non-finite iterate at iteration " + std::to_string(iters));
    const Vec zx = ax, zy = ay;
    pdhg_report rc = se.Evaluate(x.data(), y.data());
    pdhg_report ra = se.Evaluate(zx.data(), zy.data());
    double kc = Kkt(rc.primal_res, rc.dual_res, rc.gap_abs, omega);
    double ka = Kkt(ra.primal_res, ra.dual_res, ra.gap_abs, omega);
    bool take_cur = kc < ka;
    double kcand = take_cur ? kc : ka;
    const Vec cx = take_cur ? x : zx, cy = take_cur ? y : zy;
    if (EvalAndMaybeFinish(x, y, &zx, &zy)) return true;
    pdhg_eval_info info{};
    info.iteration = iters;
    info.inner_iteration = inner;
    info.restarts = restarts;
    info.omega = omega;
    info.eta = eta;
    info.kkt_candidate = kcand;
    info.kkt_loop_start = kkt_start;
    info.candidate_is_current = take_cur;
    info.original_report = last_rep;
    info.seconds = Secs();
    if (prm.restart_enabled && ShouldRestart(prm, inner, iters, kcand, kkt_start, kkt_prev)) {
      info.restarted = 1;
      double dx = 0.0, dy = 0.0;  // Restart (solver.cpp:430-446)
      for (I j = 0; j < n; ++j) { double d = cx[j] - xs[j]; dx += d * d; }
      for (I i = 0; i < m; ++i) { double d = cy[i] - ys[i]; dy += d * d; }
      omega = UpdateOmega(omega, std::sqrt(dx), std::sqrt(dy));
      x = cx;
      y = cy;
      Kx(x, kxc);
      StartAt();
      ++restarts;
    } else {
      kkt_prev = kcand;
    }
    if (prm.log_every > 0 && (info.iteration - last_log >= prm.log_every || info.iteration == 0)) {
      last_log = info.iteration;
      std::printf("iter=%lld time=%.3f rel_primal=%.3e rel_dual=%.3e rel_gap=%.3e omega=%.3e restarts=%lld\n",
                  (long long)info.iteration, info.seconds, info.original_report.rel_primal,
                  info.original_report.rel_dual, info.original_report.rel_gap, info.omega,
                  (long long)info.restarts);
    }
    if (cb && cb(&info, user) != 0) throw std::runtime_error("aborted by observer");
    return false;
  }
  void Run() {  // solver.cpp:232-267
    double on = OpNorm(k, 100, prm.seed);
    eta = on > 0.0 ? 0.9 / on : 1.0;
    omega = 1.0;
    if (se.cn > 1e-10 && se.qn > 1e-10) omega = se.cn / se.qn;
    x.assign(n, 0.0);
    for (I j = 0; j < n; ++j) x[j] = Clamp(0.0, sc.l[j], sc.u[j]);
    y.assign(m, 0.0);
    Kx(x, kxc);
    StartAt();
    if (EvalAndMaybeFinish(x, y, nullptr, nullptr)) return;
    while (true) {
      if (iters >= prm.iter_limit) { status = PDHG_ITER_LIMIT; break; }
      if (Secs() >= prm.time_limit) { status = PDHG_TIME_LIMIT; break; }
      Step();
      if (iters % prm.check_every == 0 && Check()) return;
    }
    if (!have_best) {  // UseBestSeen (solver.cpp:464-471)
      pdhg_report r;
      EvalOrig(x, y, &r);
      RecordBest(r);
    }
  }
};

Vec DeriveLambda(const Lp& p, const Vec& y) {  // kkt.cpp:127-141
  Vec lam(p.n());
  p.a.MulT(y.data(), lam.data());
  p.g.MulTAdd(1.0, y.data() + p.m1(), lam.data());
  for (I j = 0; j < p.n(); ++j) lam[j] = Proj(p.c[j] - lam[j], Cls(p.l[j], p.u[j]));
  return lam;
}

int Fail(char* err, size_t len, int code, const char* msg) {
  if (err && len) std::snprintf(err, len, "%s", msg);
  return code;
}

template <class F>
int Guard(char* err, size_t len, F&& f) {
  try {
    f();
    return PDHG_OK;
  } catch (const std::invalid_argument& e) {
    return Fail(err, len, PDHG_INVALID_ARGUMENT, e.what());
  } catch (const NumFail& e) {
    return Fail(err, len, PDHG_NUMERICAL_FAILURE, e.what());
  } catch (const std::exception& e) {
    return Fail(err, len, PDHG_ABORTED, e.what());
  }
}

struct Scaled {
  Lp orig, sc;
  Vec rs, cs;
};
Scaled Prepare(const pdhg_lp& v, const pdhg_params& prm) {
  Scaled s;
  s.orig = FromLp(v);
  Mat k = VStack(s.orig.a, s.orig.g);
  ComputeScaling(k, prm, s.rs, s.cs);
  s.sc = prm.scaling_enabled ? ApplyScaling(s.orig, s.rs, s.cs) : s.orig;
  return s;
}

}  // namespace

extern "C" {

int oracle_solve(const pdhg_lp* lp, const pdhg_params* prm, pdhg_eval_cb cb, void* user, pdhg_result* out,
                 char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    Validate(*lp);
    ValidateParams(*prm);
    auto t0 = std::chrono::steady_clock::now();
    Scaled s = Prepare(*lp, *prm);
    double scale_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    Loop loop(s.orig, s.sc, s.rs, s.cs, *prm, cb, user);
    loop.Run();
    out->status = loop.status;
    out->report = loop.best_rep;
    out->iterations = loop.iters;
    out->restarts = loop.restarts;
    out->solve_seconds = loop.Secs();
    out->scaling_seconds = scale_s;
    if (out->x) std::copy(loop.bx.begin(), loop.bx.end(), out->x);
    if (out->y) std::copy(loop.by.begin(), loop.by.end(), out->y);
    if (out->lambda) {
      Vec lam = DeriveLambda(s.orig, loop.by);
      std::copy(lam.begin(), lam.end(), out->lambda);
    }
  });
}

// Composed scales (scaling.cpp:86-91).
int oracle_scaling(const pdhg_lp* lp, const pdhg_params* prm, double* rs, double* cs, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    Scaled s = Prepare(*lp, *prm);
    std::copy(s.rs.begin(), s.rs.end(), rs);
    std::copy(s.cs.begin(), s.cs.end(), cs);
  });
}

// Scaled stacked problem (solver.cpp:227-229 on ApplyScaling's output).
int oracle_scaled(const pdhg_lp* lp, const pdhg_params* prm, double* kv, double* c, double* l, double* u, double* q,
                  char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    Scaled s = Prepare(*lp, *prm);
    Mat k = VStack(s.sc.a, s.sc.g);
    if (kv) std::copy(k.rv.begin(), k.rv.end(), kv);
    if (c) std::copy(s.sc.c.begin(), s.sc.c.end(), c);
    if (l) std::copy(s.sc.l.begin(), s.sc.l.end(), l);
    if (u) std::copy(s.sc.u.begin(), s.sc.u.end(), u);
    if (q) {
      std::copy(s.sc.b.begin(), s.sc.b.end(), q);
      std::copy(s.sc.h.begin(), s.sc.h.end(), q + s.sc.b.size());
    }
  });
}

int oracle_spmv(const pdhg_lp* lp, const pdhg_params* prm, int transpose, const double* in, double* out, char* err,
                size_t errlen) {
  return Guard(err, errlen, [&] {
    Scaled s = Prepare(*lp, *prm);
    Mat k = VStack(s.sc.a, s.sc.g);
    if (transpose) k.MulT(in, out);
    else k.Mul(in, out);
  });
}

int oracle_opnorm(const pdhg_lp* lp, const pdhg_params* prm, int iters, uint64_t seed, double* out, char* err,
                  size_t errlen) {
  return Guard(err, errlen, [&] {
    Scaled s = Prepare(*lp, *prm);
    *out = OpNorm(VStack(s.sc.a, s.sc.g), iters, seed);
  });
}

// ComputeResiduals (kkt.cpp:159-161) on the ORIGINAL problem.
int oracle_residuals(const pdhg_lp* lp, const double* x, const double* y, pdhg_report* out, char* err,
                     size_t errlen) {
  return Guard(err, errlen, [&] {
    Lp p = FromLp(*lp);
    Eval e(p);
    *out = e.Evaluate(x, y);
  });
}

// ComputeResiduals (kkt.cpp:143-145 -> ResidualEvaluator::Evaluate,
// kkt.cpp:58-118) straight on the caller's CSR view, without the CSC copy:
// for instances too large to duplicate on the host (config 5, 1e9 nnz).
// K^T y is scattered row by row, so column j accumulates its terms in
// ascending row order starting from 0.0 -- the order of the CSC that
// BuildCscFromCsr (sparse_matrix.cpp:71-88) builds -- and the G part is
// completed before it is added (MultiplyTransposeAdd, sparse_matrix.cpp:153).
// Bit-identical to oracle_residuals / the reference for a valid CSR (rows
// sorted, no duplicates); tests/test_oracle.py pins it.
int oracle_residuals_view(const pdhg_lp* lp, const double* x, const double* y, pdhg_report* out, char* err,
                          size_t errlen) {
  return Guard(err, errlen, [&] {
    const pdhg_lp& v = *lp;
    const I n = v.n, m1 = v.a.rows, m2 = v.g.rows;
    auto rowsum = [](const pdhg_csr& a, I r, const double* xx) {
      double acc = 0.0;
      for (int64_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) acc += a.values[k] * xx[a.col_idx[k]];
      return acc;
    };
    double ps = 0.0;
    for (I i = 0; i < m1; ++i) {
      const double d = rowsum(v.a, i, x) - v.b[i];
      ps += d * d;
    }
    for (I i = 0; i < m2; ++i) {
      const double d = std::max(v.h[i] - rowsum(v.g, i, x), 0.0);
      ps += d * d;
    }
    Vec kty(n, 0.0), ktg(n, 0.0);
    for (I i = 0; i < m1; ++i)
      for (int64_t k = v.a.row_ptr[i]; k < v.a.row_ptr[i + 1]; ++k) kty[v.a.col_idx[k]] += v.a.values[k] * y[i];
    for (I i = 0; i < m2; ++i)
      for (int64_t k = v.g.row_ptr[i]; k < v.g.row_ptr[i + 1]; ++k)
        ktg[v.g.col_idx[k]] += v.g.values[k] * y[m1 + i];
    for (I j = 0; j < n; ++j) kty[j] += 1.0 * ktg[j];
    pdhg_report r{};
    r.primal_res = std::sqrt(ps);
    double ds = 0.0, bt = 0.0;
    for (I j = 0; j < n; ++j) {
      const double red = v.c[j] - kty[j];
      const double lam = Proj(red, Cls(v.l[j], v.u[j]));
      const double d = red - lam;
      ds += d * d;
      if (lam > 0.0) bt += v.l[j] * lam;
      else if (lam < 0.0) bt += v.u[j] * lam;
    }
    r.dual_res = std::sqrt(ds);
    double po = v.objective_offset;
    for (I j = 0; j < n; ++j) po += v.c[j] * x[j];
    double dob = v.objective_offset + bt;
    for (I i = 0; i < m1; ++i) dob += v.b[i] * y[i];
    for (I i = 0; i < m2; ++i) dob += v.h[i] * y[m1 + i];
    const double cn = Norm2(v.c, n);
    double qs = 0.0;
    for (I i = 0; i < m1; ++i) qs += v.b[i] * v.b[i];
    for (I i = 0; i < m2; ++i) qs += v.h[i] * v.h[i];
    const double qn = std::sqrt(qs);
    r.primal_obj = po;
    r.dual_obj = dob;
    r.gap_abs = std::abs(dob - po);
    r.rel_primal = r.primal_res / (1.0 + qn);
    r.rel_dual = r.dual_res / (1.0 + cn);
    r.rel_gap = r.gap_abs / (1.0 + std::abs(dob) + std::abs(po));
    *out = r;
  });
}

// PrimalStep / DualStep (solver.cpp:112-154) on the unscaled problem.
int oracle_primal_step(const pdhg_lp* lp, const double* x, const double* y, double eta, double omega, double* out,
                       char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    Lp p = FromLp(*lp);
    Vec kty(p.n());
    p.a.MulT(y, kty.data());
    p.g.MulTAdd(1.0, y + p.m1(), kty.data());
    const double st = eta / omega;
    for (I j = 0; j < p.n(); ++j) out[j] = Clamp(x[j] - st * (p.c[j] - kty[j]), p.l[j], p.u[j]);
  });
}

int oracle_dual_step(const pdhg_lp* lp, const double* xn, const double* xo, const double* y, double eta,
                     double omega, double* out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    Lp p = FromLp(*lp);
    Vec ext(p.n()), kx(p.m1() + p.m2());
    for (I j = 0; j < p.n(); ++j) ext[j] = 2.0 * xn[j] - xo[j];
    p.a.Mul(ext.data(), kx.data());
    p.g.Mul(ext.data(), kx.data() + p.m1());
    const double st = eta * omega;
    for (I i = 0; i < p.m1(); ++i) out[i] = y[i] + st * (p.b[i] - kx[i]);
    for (I i = 0; i < p.m2(); ++i) out[p.m1() + i] = std::max(y[p.m1() + i] + st * (p.h[i] - kx[p.m1() + i]), 0.0);
  });
}

}  // extern "C"
