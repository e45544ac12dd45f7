// Epilogue ops for the tile engine: each op fuses one reference loop with
// the SpMV that feeds it. Reference loops cited per op. All arithmetic is
// compiled with -fmad=false so every `a * b + c` rounds twice, as on the
// reference's x86-64 baseline build (no FMA contraction).
//
// Per-segment epilogue operands come from `operand(k)` arrays that the engine
// stages by TMA for the tile's whole segment range (`staged`); `prefetch`
// reads the same operands from global memory for the rare segments finished
// outside their own tile. The epilogue itself only stores.
#pragma once

#include "engine.cuh"

namespace pdhg {

// ---------------------------------------------------------------- plain SpMV
// y = M x (sparse_matrix.cpp:114-125 / 127-138).
struct OpSpmv {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  static constexpr bool kUniform = true;
  using Pre = Nil;
  const double* x;
  double* y;
  __device__ void map(int32_t j, double v, double (&p)[1]) const { p[0] = v * x[j]; }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 0;
  __device__ const double* operand(int) const { return nullptr; }
  __device__ Pre staged(int32_t, const double*, int) const { return {}; }
  __device__ Pre prefetch(int32_t) const { return {}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre&, double*) const { y[s] = a[0]; }
};

// ------------------------------------------------------------ power iteration
// EstimateOpNorm (solver.cpp:84-110): the reference stores v / ||v|| and then
// multiplies; we gather u[j] / norm, the same IEEE division per element.
// kSumSq: also accumulate sum(y^2) for the next normalisation.
template <bool kSumSq>
struct OpPowerStep {
  static constexpr int kRhs = 1, kRed = kSumSq ? 1 : 0;
  static constexpr bool kMax = false;
  static constexpr bool kUniform = true;
  static constexpr bool kPdl = true;  // no prologue operands; gathers and pw_norm after the wait
  using Pre = Nil;
  const double* x;
  const Scalars* sc;  // pw_norm divides the gathered operand
  int divide;
  double* y;
  __device__ void map(int32_t j, double v, double (&p)[1]) const {
    p[0] = divide ? v * (x[j] / sc->pw_norm) : v * x[j];
  }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 0;
  __device__ const double* operand(int) const { return nullptr; }
  __device__ Pre staged(int32_t, const double*, int) const { return {}; }
  __device__ Pre prefetch(int32_t) const { return {}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre&, double* red) const {
    y[s] = a[0];
    if constexpr (kSumSq) red[0] += a[0] * a[0];
  }
};

// ------------------------------------------------------------------ scaling
// Ruiz sweep norms (scaling.cpp:49-68 via RowInfNorms/ColInfNorms,
// sparse_matrix.cpp:166-184): d = 1/sqrt(max|v|) (1 for empty), scale *= d.
struct OpInfNormScale {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = true;
  using Pre = Nil;
  double* d;      // this sweep's factor
  double* scale;  // accumulated Ruiz scale
  __device__ void map(int32_t, double v, double (&p)[1]) const { p[0] = fabs(v); }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 0;
  __device__ const double* operand(int) const { return nullptr; }
  __device__ Pre staged(int32_t, const double*, int) const { return {}; }
  __device__ Pre prefetch(int32_t) const { return {}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre&, double*) const {
    const double f = a[0] > 0.0 ? 1.0 / sqrt(a[0]) : 1.0;
    d[s] = f;
    scale[s] *= f;
  }
};

// Pock-Chambolle (scaling.cpp:70-84 via RowPowerSums/ColPowerSums,
// sparse_matrix.cpp:186-204): scale *= 1/sqrt(sum |v|^p). std::pow is
// special-cased for p in {0, 1, 2} so the common alpha=1 path is exact.
struct OpPowerSumScale {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  using Pre = Nil;
  double pw;
  int mode;  // 0: |v|^0 = 1, 1: |v|, 2: v*v, 3: pow
  double* scale;
  __device__ void map(int32_t, double v, double (&p)[1]) const {
    const double a = fabs(v);
    p[0] = mode == 1 ? a : (mode == 2 ? a * a : (mode == 0 ? 1.0 : pow(a, pw)));
  }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 0;
  __device__ const double* operand(int) const { return nullptr; }
  __device__ Pre staged(int32_t, const double*, int) const { return {}; }
  __device__ Pre prefetch(int32_t) const { return {}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre&, double*) const {
    if (a[0] > 0.0) scale[s] *= 1.0 / sqrt(a[0]);
  }
};

// Raw per-segment reductions (sparse_matrix.cpp:166-204): max |v| (kMax) or
// sum |v|^p in storage order, p special-cased for {0, 1, 2} like
// OpPowerSumScale (std::pow is exact there; other p use the device pow).
template <bool kInf>
struct OpRawNorm {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = kInf;
  using Pre = Nil;
  double pw;
  int mode;  // power sums: 0 |v|^0, 1 |v|, 2 v*v, 3 pow
  double* out;
  __device__ void map(int32_t, double v, double (&p)[1]) const {
    const double a = fabs(v);
    if constexpr (kInf) p[0] = a;
    else p[0] = mode == 1 ? a : (mode == 2 ? a * a : (mode == 0 ? 1.0 : pow(a, pw)));
  }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 0;
  __device__ const double* operand(int) const { return nullptr; }
  __device__ Pre staged(int32_t, const double*, int) const { return {}; }
  __device__ Pre prefetch(int32_t) const { return {}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre&, double*) const { out[s] = a[0]; }
};

// --------------------------------------------------------- PDHG step kernels
// K-CSC: kty = K^T y, x+ = proj_[l,u](x - (eta/omega)(c - kty)), running
// average of x (solver.cpp:285-290, RunningAverage::Add x-half :159).
// kBnd: bit 0 -- every scaled lower bound equals sc->lb, bit 1 -- every upper
// bound equals sc->ub (e.g. x >= 0: l_s = 0 / cs = 0, u_s = inf / cs = inf),
// so those arrays are never streamed (16 of the 56 vector bytes per column).
template <bool kAdapt, int kBnd = 0>
struct OpPrimal {
  static constexpr int kRhs = 1, kRed = kAdapt ? 1 : 0;
  static constexpr bool kMax = false;
  static constexpr bool kL = !(kBnd & 1), kU = !(kBnd & 2);  // streamed?
  static constexpr bool kUniform = true;                     // per-iteration: specialise
  static constexpr bool kPdl = true;                         // programmatic dependent launch
  static constexpr int kIL = 2, kIU = 2 + kL, kIB = 2 + kL + kU;  // operand slots
  struct Pre {
    double x, c, l, u, xbar, w, step;
  };
  const double* y;  // current dual
  const double* x;  // current primal
  double* xn;       // next primal
  double* xbar;     // running average
  const double* c;
  const double* l;
  const double* u;
  const Scalars* sc;
  int j_in_block;
  // Pipelined loop only: &sc->halt, so a block queued behind a halting check
  // is discarded. Null elsewhere -- no load of the flag ahead of the pass.
  const int32_t* halt = nullptr;
  __device__ bool skip() const { return halt && *halt != 0; }
  __device__ void map(int32_t i, double v, double (&p)[1]) const { p[0] = v * y[i]; }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 3 + kL + kU;
  __device__ const double* operand(int k) const {
    if (k == 0) return x;
    if (k == 1) return c;
    if (kL && k == kIL) return l;
    if (kU && k == kIU) return u;
    return xbar;
  }
  __device__ Pre staged(int32_t, const double* st, int ld) const {
    Pre p;
    p.w = sc->inner_base + static_cast<double>(j_in_block);
    p.step = sc->step_p;
    p.x = st[0];
    p.c = st[ld];
    p.l = kL ? st[kIL * ld] : sc->lb;
    p.u = kU ? st[kIU * ld] : sc->ub;
    p.xbar = (p.w == 0.0) ? 0.0 : st[kIB * ld];
    return p;
  }
  __device__ Pre prefetch(int32_t s) const {
    // The per-segment loads go out first (the average speculatively: it is
    // only used when w > 0), the solver scalars after them.
    Pre p;
    p.x = x[s];
    p.c = c[s];
    if constexpr (kL) p.l = l[s];
    if constexpr (kU) p.u = u[s];
    const double xb = xbar[s];
    p.w = sc->inner_base + static_cast<double>(j_in_block);
    p.step = sc->step_p;
    if constexpr (!kL) p.l = sc->lb;
    if constexpr (!kU) p.u = sc->ub;
    p.xbar = (p.w == 0.0) ? 0.0 : xb;  // Reset() zeroes the average
    return p;
  }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre& p, double* red) const {
    const double xv = clamp_ref(p.x - p.step * (p.c - a[0]), p.l, p.u);
    xn[s] = xv;
    xbar[s] = (p.w * p.xbar + xv) / (p.w + 1.0);
    if constexpr (kAdapt) {
      const double d = xv - p.x;  // AdaptStepSize (solver.cpp:312-315)
      red[0] += d * d;
    }
  }
};

// K-CSR: kx+ = K x+, y+ = proj_Y(y + eta*omega (q - (2 kx+ - kx))), running
// average of y (solver.cpp:292-298, :160). The reflected point 2x+ - x is
// never formed: linearity gives K(2x+ - x) = 2 kx+ - kx (solver.cpp:296).
template <bool kAdapt>
struct OpDual {
  static constexpr int kRhs = 1, kRed = kAdapt ? 2 : 0;
  static constexpr bool kMax = false;
  static constexpr bool kUniform = true;
  static constexpr bool kPdl = true;
  static constexpr bool kSplit = !kAdapt;  // gather-window split of class S (engine.cuh launch_class_s)
  struct Pre {
    double kx, y, q, ybar, w, step;
  };
  const double* xn;  // next primal (gathered)
  const double* y;
  double* yn;
  double* ybar;
  const double* kx;  // K x (current)
  double* kxn;       // K x+ (next)
  const double* q;
  RowKind rk;  // equality rows (permuted order)
  const Scalars* sc;
  int j_in_block;
  const int32_t* halt = nullptr;  // as OpPrimal::halt
  __device__ bool skip() const { return halt && *halt != 0; }
  __device__ void map(int32_t j, double v, double (&p)[1]) const { p[0] = v * xn[j]; }
  __device__ double gather(int32_t j) const { return xn[j]; }
  __device__ void prod(double v, double g, double (&p)[1]) const { p[0] = v * g; }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 4;
  __device__ const double* operand(int k) const {
    const double* a[4] = {kx, y, q, ybar};
    return a[k];
  }
  __device__ Pre staged(int32_t, const double* st, int ld) const {
    Pre p;
    p.w = sc->inner_base + static_cast<double>(j_in_block);
    p.step = sc->step_d;
    p.kx = st[0];
    p.y = st[ld];
    p.q = st[2 * ld];
    p.ybar = (p.w == 0.0) ? 0.0 : st[3 * ld];
    return p;
  }
  __device__ Pre prefetch(int32_t s) const {
    Pre p;  // per-segment loads first (the average speculatively), scalars after
    p.kx = kx[s];
    p.y = y[s];
    p.q = q[s];
    const double yb = ybar[s];
    p.w = sc->inner_base + static_cast<double>(j_in_block);
    p.step = sc->step_d;
    p.ybar = (p.w == 0.0) ? 0.0 : yb;
    return p;
  }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre& p, double* red) const {
    const double v = p.y + p.step * (p.q - (2.0 * a[0] - p.kx));
    const double yv = rk.eq(s) ? v : max0_ref(v);
    yn[s] = yv;
    kxn[s] = a[0];
    ybar[s] = (p.w * p.ybar + yv) / (p.w + 1.0);
    if constexpr (kAdapt) {
      const double d = yv - p.y;  // AdaptStepSize (solver.cpp:316-320)
      red[0] += d * d;
      red[1] += d * (a[0] - p.kx);
    }
  }
};

// ------------------------------------------------------------- check passes
// Reduction slots of the check (per point P in {cur, avg}).
enum CheckRow { kPrS = 0, kPrO, kQyS, kQyO, kDy2, kRowPer };  // + 1 nonfinite-y count
enum CheckCol { kDuS = 0, kDuO, kBdS, kBdO, kCxS, kCxO, kDx2, kColPer };  // + 1 nonfinite-x
constexpr int kRowRed = 2 * kRowPer + 1;
constexpr int kColRed = 2 * kColPer + 1;

// Row side of ResidualEvaluator::Evaluate (kkt.cpp:58-76, :104-109) for the
// current point and the running average at once, in the scaled space
// (restart candidate KKT_omega, solver.cpp:396-397) and the original space
// (termination, solver.cpp:330-339) -- the latter through
// K_orig x_orig = D_r^{-1} (K_s x_s). Also dy for the primal-weight update
// (solver.cpp:437-440) and the finite test of y (solver.cpp:391).
struct OpCheckRow {
  static constexpr int kRhs = 1, kRed = kRowRed;
  static constexpr bool kMax = false;
  static constexpr bool kUniform = true;
  struct Pre {
    double kx, y, yb, y0, qs, qo, r;
  };
  const double* xbar;  // gathered: K xbar
  double* kx_avg;      // out
  const double* kx_cur;
  const double* y_cur;
  const double* ybar;
  const double* y_start;
  const double* q_s;
  const double* q_o;
  const double* rs;
  RowKind rk;  // equality rows (permuted order)
  const Scalars* sc;  // null outside the pipelined loop
  __device__ bool skip() const { return sc && sc->halt != 0; }
  __device__ void map(int32_t j, double v, double (&p)[1]) const { p[0] = v * xbar[j]; }
  static constexpr int kOcc = 2;
  static constexpr int kOps = 7;
  __device__ const double* operand(int k) const {
    const double* a[7] = {kx_cur, y_cur, ybar, y_start, q_s, q_o, rs};
    return a[k];
  }
  __device__ Pre staged(int32_t, const double* st, int ld) const {
    return {st[0], st[ld], st[2 * ld], st[3 * ld], st[4 * ld], st[5 * ld], st[6 * ld]};
  }
  __device__ Pre prefetch(int32_t s) const {
    return {kx_cur[s], y_cur[s], ybar[s], y_start[s], q_s[s], q_o[s], rs[s]};
  }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre& p, double* red) const {
    kx_avg[s] = a[0];
#pragma unroll
    for (int P = 0; P < 2; ++P) {
      const double kx = P == 0 ? p.kx : a[0];
      const double yv = P == 0 ? p.y : p.yb;
      double* o = red + P * kRowPer;
      const double es = rk.eq(s) ? kx - p.qs : max0_ref(p.qs - kx);
      o[kPrS] += es * es;
      const double kxo = kx / p.r;
      const double eo = rk.eq(s) ? kxo - p.qo : max0_ref(p.qo - kxo);
      o[kPrO] += eo * eo;
      o[kQyS] += p.qs * yv;
      o[kQyO] += p.qo * (yv * p.r);
      const double dy = yv - p.y0;
      o[kDy2] += dy * dy;
    }
    if (!isfinite(p.y)) red[2 * kRowPer] += 1.0;
  }
};

// Column side (kkt.cpp:78-103): lambda = proj(c - K'y), dual residual, bound
// term, c'x for both points and both spaces; dx for the primal weight
// (solver.cpp:433-436); finite test of x (solver.cpp:391). Two gathered
// operands: K^T [y_cur, ybar] from one pass over the matrix.
// kUB: every column shares its scaled and original bounds (x >= 0: l_s = l_o = 0,
// u_s = u_o = inf), carried in lb/ub instead of four streamed arrays.
template <bool kUB = false>
struct OpCheckCol {
  static constexpr int kRhs = 2, kRed = kColRed;
  static constexpr bool kMax = false;
  static constexpr bool kUniform = true;
  struct Pre {
    double x, xb, x0, cS, lS, uS, cO, lO, uO, f;
  };
  const double* y_cur;
  const double* ybar;
  const double* x_cur;
  const double* xbar;
  const double* x_start;
  const double* c_s;
  const double* l_s;
  const double* u_s;
  const double* c_o;
  const double* l_o;
  const double* u_o;
  const double* cs;
  const Scalars* sc;  // null outside the pipelined loop
  double lb = 0.0, ub = 0.0;  // kUB: the common bounds (both spaces)
  __device__ bool skip() const { return sc && sc->halt != 0; }
  __device__ void map(int32_t i, double v, double (&p)[2]) const {
    p[0] = v * y_cur[i];
    p[1] = v * ybar[i];
  }
  static constexpr int kOcc = 2;
  static constexpr int kOps = kUB ? 6 : 10;
  __device__ const double* operand(int k) const {
    if constexpr (kUB) {
      const double* a[6] = {x_cur, xbar, x_start, c_s, c_o, cs};
      return a[k];
    } else {
      const double* a[10] = {x_cur, xbar, x_start, c_s, l_s, u_s, c_o, l_o, u_o, cs};
      return a[k];
    }
  }
  __device__ Pre staged(int32_t, const double* st, int ld) const {
    if constexpr (kUB)
      return {st[0], st[ld], st[2 * ld], st[3 * ld], lb, ub, st[4 * ld], lb, ub, st[5 * ld]};
    else
      return {st[0], st[ld], st[2 * ld], st[3 * ld], st[4 * ld], st[5 * ld], st[6 * ld], st[7 * ld], st[8 * ld],
              st[9 * ld]};
  }
  __device__ Pre prefetch(int32_t s) const {
    if constexpr (kUB)
      return {x_cur[s], xbar[s], x_start[s], c_s[s], lb, ub, c_o[s], lb, ub, cs[s]};
    else
      return {x_cur[s], xbar[s], x_start[s], c_s[s], l_s[s], u_s[s], c_o[s], l_o[s], u_o[s], cs[s]};
  }
  __device__ void finish(int32_t s, const double (&a)[2], const Pre& p, double* red) const {
    const int cls = bound_class(p.lO, p.uO);
#pragma unroll
    for (int P = 0; P < 2; ++P) {
      const double kty = a[P];
      const double xv = P == 0 ? p.x : p.xb;
      double* o = red + P * kColPer;
      const double rS = p.cS - kty;
      const double lamS = project_reduced(rS, cls);
      const double dS = rS - lamS;
      o[kDuS] += dS * dS;
      if (lamS > 0.0) o[kBdS] += p.lS * lamS;
      else if (lamS < 0.0) o[kBdS] += p.uS * lamS;
      const double rO = p.cO - kty / p.f;
      const double lamO = project_reduced(rO, cls);
      const double dO = rO - lamO;
      o[kDuO] += dO * dO;
      if (lamO > 0.0) o[kBdO] += p.lO * lamO;
      else if (lamO < 0.0) o[kBdO] += p.uO * lamO;
      o[kCxS] += p.cS * xv;
      o[kCxO] += p.cO * (xv * p.f);
      const double dx = xv - p.x0;
      o[kDx2] += dx * dx;
    }
    if (!isfinite(p.x)) red[2 * kColPer] += 1.0;
  }
};

// DeriveLambda (kkt.cpp:127-141) for the returned y, original space.
struct OpLambda {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  static constexpr bool kUniform = true;
  struct Pre {
    double c, l, u, f;
  };
  const double* y_s;  // scaled dual
  const double* c_o;
  const double* l_o;
  const double* u_o;
  const double* cs;
  double* lam;
  __device__ void map(int32_t i, double v, double (&p)[1]) const { p[0] = v * y_s[i]; }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 4;
  __device__ const double* operand(int k) const {
    const double* a[4] = {c_o, l_o, u_o, cs};
    return a[k];
  }
  __device__ Pre staged(int32_t, const double* st, int ld) const {
    return {st[0], st[ld], st[2 * ld], st[3 * ld]};
  }
  __device__ Pre prefetch(int32_t s) const { return {c_o[s], l_o[s], u_o[s], cs[s]}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre& p, double*) const {
    lam[s] = project_reduced(p.c - a[0] / p.f, bound_class(p.l, p.u));
  }
};

// PrimalStep / DualStep unit exports (solver.cpp:112-154) on an unscaled K.
struct OpUnitPrimal {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  struct Pre {
    double x, c, l, u;
  };
  const double* y;
  const double* x;
  const double* c;
  const double* l;
  const double* u;
  double step;  // eta / omega
  double* out;
  __device__ void map(int32_t i, double v, double (&p)[1]) const { p[0] = v * y[i]; }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 4;
  __device__ const double* operand(int k) const {
    const double* a[4] = {x, c, l, u};
    return a[k];
  }
  __device__ Pre staged(int32_t, const double* st, int ld) const {
    return {st[0], st[ld], st[2 * ld], st[3 * ld]};
  }
  __device__ Pre prefetch(int32_t s) const { return {x[s], c[s], l[s], u[s]}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre& p, double*) const {
    out[s] = clamp_ref(p.x - step * (p.c - a[0]), p.l, p.u);
  }
};

struct OpUnitDual {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  struct Pre {
    double y, q;
  };
  const double* ext;  // 2 x_new - x_old
  const double* y;
  const double* q;
  RowKind rk;  // equality rows (permuted order)
  double step;  // eta * omega
  double* out;
  __device__ void map(int32_t j, double v, double (&p)[1]) const { p[0] = v * ext[j]; }
  static constexpr int kOcc = 5;
  static constexpr int kOps = 2;
  __device__ const double* operand(int k) const {
    const double* a[2] = {y, q};
    return a[k];
  }
  __device__ Pre staged(int32_t, const double* st, int ld) const { return {st[0], st[ld]}; }
  __device__ Pre prefetch(int32_t s) const { return {y[s], q[s]}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre& p, double*) const {
    const double v = p.y + step * (p.q - a[0]);
    out[s] = rk.eq(s) ? v : max0_ref(v);
  }
};

}  // namespace pdhg
