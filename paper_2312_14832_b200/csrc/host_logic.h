// Host-side decision logic of the solve loop, shared by the session and the
// C-ABI exports. Restated from the reference (file:line per function).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>

#include "../../include/pdhg.h"

#if defined(__CUDACC__)
#define PDHG_HD __host__ __device__
#else
#define PDHG_HD
#endif

namespace pdhg {

// LpProblem::Validate (lp_problem.cpp:22-58): same checks, same messages,
// same precedence (NaN in c, b, h; then infinite c; then the first index
// with a NaN or crossed bound). The element scans run on up to 8 threads for
// large n -- each chunk reports flags / its first bad index, merged in
// index order -- since they sit in front of every one-shot solve.
struct LpScan {
  bool nan_c = false, inf_c = false;
  int64_t bad_bound = -1;  // first index with a NaN or crossed bound
};

inline void ScanLp(const pdhg_lp& lp, int64_t b, int64_t e, LpScan* out) {
  bool nan_c = false, inf_c = false;
  for (int64_t i = b; i < e; ++i) {
    nan_c |= std::isnan(lp.c[i]);
    inf_c |= std::isinf(lp.c[i]);
  }
  out->nan_c = nan_c;
  out->inf_c = inf_c;
  for (int64_t i = b; i < e; ++i)
    if (std::isnan(lp.l[i]) || std::isnan(lp.u[i]) || lp.l[i] > lp.u[i]) {
      out->bad_bound = i;
      break;
    }
}

inline void ValidateLpHost(const pdhg_lp& lp) {
  auto bad = [](const std::string& m) { throw std::invalid_argument(m); };
  const int64_t n = lp.n;
  if (n < 0 || lp.a.rows < 0 || lp.g.rows < 0) bad("negative matrix dimension");
  if (lp.a.cols != n || lp.g.cols != n) bad("matrix column count does not match c");
  if ((lp.a.rows && !lp.a.row_ptr) || (lp.g.rows && !lp.g.row_ptr)) bad("missing row_ptr");
  if ((n && (!lp.c || !lp.l || !lp.u)) || (lp.a.rows && !lp.b) || (lp.g.rows && !lp.h)) bad("missing vector");
  const int threads = n >= (int64_t(1) << 18)
                          ? static_cast<int>(std::min<unsigned>(8, std::max(1u, std::thread::hardware_concurrency())))
                          : 1;
  std::vector<LpScan> part(threads);
  {
    std::vector<std::thread> pool;
    const int64_t per = (n + threads - 1) / threads;
    for (int t = 1; t < threads; ++t)
      pool.emplace_back(ScanLp, std::cref(lp), std::min(n, t * per), std::min(n, (t + 1) * per), &part[t]);
    ScanLp(lp, 0, std::min(n, per), &part[0]);
    for (auto& th : pool) th.join();
  }
  LpScan all;
  for (const LpScan& p : part) {
    all.nan_c |= p.nan_c;
    all.inf_c |= p.inf_c;
    if (all.bad_bound < 0) all.bad_bound = p.bad_bound;
  }
  if (all.nan_c) bad("NaN in c");
  for (int64_t i = 0; i < lp.a.rows; ++i)
    if (std::isnan(lp.b[i])) bad("NaN in b");
  for (int64_t i = 0; i < lp.g.rows; ++i)
    if (std::isnan(lp.h[i])) bad("NaN in h");
  if (all.inf_c) bad("infinite entry in c");
  if (all.bad_bound >= 0) {
    const int64_t i = all.bad_bound;
    if (std::isnan(lp.l[i]) || std::isnan(lp.u[i])) bad("NaN bound");
    bad("crossed bounds: l > u at index " + std::to_string(i));
  }
}

// KktError (kkt.cpp:153-157).
// The decision helpers below are PDHG_HD: the pipelined loop evaluates them on
// the device (csrc/decide.cuh) with the same IEEE operations (sqrt, fabs,
// compares; no FMA on either side), hence bit-identical decisions.
PDHG_HD inline double KktError(double p, double d, double g, double w) {
  return sqrt(w * w * p * p + d * d / (w * w) + g * g);
}
PDHG_HD inline double Kkt1(const pdhg_report& r) { return KktError(r.primal_res, r.dual_res, r.gap_abs, 1.0); }

// CheckTermination (kkt.cpp:147-151).
PDHG_HD inline bool Terminated(const pdhg_report& r, double eps) {
  return r.rel_primal <= eps && r.rel_dual <= eps && r.rel_gap <= eps;
}

// ShouldRestart (solver.cpp:178-189): sufficient decay; necessary decay with
// no local progress; long inner loop.
PDHG_HD inline bool ShouldRestartV(double suff, double nec, double frac, int64_t t, int64_t k, double cand,
                                    double start, double prev) {
  if (cand <= suff * start) return true;
  if (cand <= nec * start && cand > prev) return true;
  return static_cast<double>(t) >= frac * static_cast<double>(k);
}
inline bool ShouldRestart(const pdhg_params& p, int64_t t, int64_t k, double cand, double start, double prev) {
  return ShouldRestartV(p.sufficient_decay, p.necessary_decay, p.long_loop_frac, t, k, cand, start, prev);
}

// UpdatePrimalWeight (solver.cpp:191-196).
inline double UpdatePrimalWeight(double w, double dx, double dy) {
  constexpr double kMin = 1e-10;
  if (dx <= kMin || dy <= kMin) return w;
  return std::exp(0.5 * std::log(dy / dx) + 0.5 * std::log(w));
}

// ResidualReport from reduced sums (kkt.cpp:80-118).
PDHG_HD inline pdhg_report MakeReport(double pr2, double du2, double bound, double cx, double qy, double off,
                                      double qn, double cn) {
  pdhg_report r{};
  r.primal_res = sqrt(pr2);
  r.dual_res = sqrt(du2);
  r.primal_obj = off + cx;
  r.dual_obj = off + bound + qy;
  r.gap_abs = fabs(r.dual_obj - r.primal_obj);
  r.rel_primal = r.primal_res / (1.0 + qn);
  r.rel_dual = r.dual_res / (1.0 + cn);
  r.rel_gap = r.gap_abs / (1.0 + fabs(r.dual_obj) + fabs(r.primal_obj));
  return r;
}

// Contiguous block partition of `nseg` segments (rows or columns, original
// order) into `parts` blocks balanced by W(s) = ptr[s] + seg_weight * s (the
// nonzeros plus a per-segment charge for the vector traffic): block b ends at
// the smallest s with W(s) * parts >= (b + 1) * W(nseg). Every rank computes
// it from the same ptr array, so the split needs no communication.
template <class P>
inline void BalancedBlocks(const P* ptr, int64_t nseg, int parts, int64_t seg_weight, int64_t* begin) {
  const auto W = [&](int64_t s) { return static_cast<long double>(ptr[s]) + static_cast<long double>(seg_weight) * s; };
  const long double total = W(nseg);
  begin[0] = 0;
  for (int b = 1; b < parts; ++b) {
    const long double target = total * b;
    int64_t lo = begin[b - 1], hi = nseg;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (W(mid) * parts >= target) hi = mid;
      else lo = mid + 1;
    }
    begin[b] = lo;
  }
  begin[parts] = nseg;
}

}  // namespace pdhg
