// Epilogue ops for the tile engine: each op fuses one reference loop with
// the SpMV that feeds it. Reference loops cited per op. All arithmetic is
// compiled with -fmad=false so every `a * b + c` rounds twice, as on the
// reference's x86-64 baseline build (no FMA contraction).
#pragma once

#include "tile_spmv.cuh"

namespace pdhg {

// ---------------------------------------------------------------- plain SpMV
// y = M x (sparse_matrix.cpp:114-125 / 127-138).
struct OpSpmv {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  const double* x;
  double* y;
  __device__ void map(int32_t j, double v, double (&p)[1]) const { p[0] = v * x[j]; }
  __device__ void finish(int32_t s, const double (&a)[1], double*) const { y[s] = a[0]; }
};

// ------------------------------------------------------------ power iteration
// EstimateOpNorm (solver.cpp:84-110): the reference stores v / ||v|| and then
// multiplies; we gather u[j] / norm, the same IEEE division per element.
// kSumSq: also accumulate sum(y^2) for the next normalisation.
template <bool kSumSq>
struct OpPowerStep {
  static constexpr int kRhs = 1, kRed = kSumSq ? 1 : 0;
  static constexpr bool kMax = false;
  const double* x;
  const Scalars* sc;  // pw_norm divides the gathered operand (1.0 for none)
  int divide;
  double* y;
  __device__ void map(int32_t j, double v, double (&p)[1]) const {
    p[0] = divide ? v * (x[j] / sc->pw_norm) : v * x[j];
  }
  __device__ void finish(int32_t s, const double (&a)[1], double* red) const {
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
  double* d;      // this sweep's factor
  double* scale;  // accumulated Ruiz scale
  __device__ void map(int32_t, double v, double (&p)[1]) const { p[0] = fabs(v); }
  __device__ void finish(int32_t s, const double (&a)[1], double*) const {
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
  double pw;
  int mode;  // 0: |v|^0 = 1, 1: |v|, 2: v*v, 3: pow
  double* scale;
  __device__ void map(int32_t, double v, double (&p)[1]) const {
    const double a = fabs(v);
    p[0] = mode == 1 ? a : (mode == 2 ? a * a : (mode == 0 ? 1.0 : pow(a, pw)));
  }
  __device__ void finish(int32_t s, const double (&a)[1], double*) const {
    if (a[0] > 0.0) scale[s] *= 1.0 / sqrt(a[0]);
  }
};

// --------------------------------------------------------- PDHG step kernels
// K-CSC: kty = K^T y, x+ = proj_[l,u](x - (eta/omega)(c - kty)), running
// average of x (solver.cpp:285-290, RunningAverage::Add x-half :159).
template <bool kAdapt>
struct OpPrimal {
  static constexpr int kRhs = 1, kRed = kAdapt ? 1 : 0;
  static constexpr bool kMax = false;
  const double* y;  // current dual
  const double* x;  // current primal
  double* xn;       // next primal
  double* xbar;     // running average
  const double* c;
  const double* l;
  const double* u;
  const Scalars* sc;
  int j_in_block;
  __device__ void map(int32_t i, double v, double (&p)[1]) const { p[0] = v * y[i]; }
  __device__ void finish(int32_t s, const double (&a)[1], double* red) const {
    const double step = sc->eta / sc->omega;
    const double xo = x[s];
    const double xv = clamp_ref(xo - step * (c[s] - a[0]), l[s], u[s]);
    xn[s] = xv;
    const double w = sc->inner_base + static_cast<double>(j_in_block);
    const double xb = (w == 0.0) ? 0.0 : xbar[s];  // Reset() zeroes the average
    xbar[s] = (w * xb + xv) / (w + 1.0);
    if constexpr (kAdapt) {
      const double d = xv - xo;  // AdaptStepSize (solver.cpp:312-315)
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
  const double* xn;  // next primal (gathered)
  const double* y;
  double* yn;
  double* ybar;
  const double* kx;  // K x (current)
  double* kxn;       // K x+ (next)
  const double* q;
  int32_t m1;
  const Scalars* sc;
  int j_in_block;
  __device__ void map(int32_t j, double v, double (&p)[1]) const { p[0] = v * xn[j]; }
  __device__ void finish(int32_t s, const double (&a)[1], double* red) const {
    const double step = sc->eta * sc->omega;
    const double k0 = kx[s];
    const double yo = y[s];
    const double v = yo + step * (q[s] - (2.0 * a[0] - k0));
    const double yv = s < m1 ? v : max0_ref(v);
    yn[s] = yv;
    kxn[s] = a[0];
    const double w = sc->inner_base + static_cast<double>(j_in_block);
    const double yb = (w == 0.0) ? 0.0 : ybar[s];
    ybar[s] = (w * yb + yv) / (w + 1.0);
    if constexpr (kAdapt) {
      const double d = yv - yo;  // AdaptStepSize (solver.cpp:316-320)
      red[0] += d * d;
      red[1] += d * (a[0] - k0);
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
  const double* xbar;  // gathered: K xbar
  double* kx_avg;      // out
  const double* kx_cur;
  const double* y_cur;
  const double* ybar;
  const double* y_start;
  const double* q_s;
  const double* q_o;
  const double* rs;
  int32_t m1;
  __device__ void map(int32_t j, double v, double (&p)[1]) const { p[0] = v * xbar[j]; }
  __device__ void finish(int32_t s, const double (&a)[1], double* red) const {
    kx_avg[s] = a[0];
    const double qs = q_s[s], qo = q_o[s], r = rs[s], ys0 = y_start[s];
#pragma unroll
    for (int P = 0; P < 2; ++P) {
      const double kx = P == 0 ? kx_cur[s] : a[0];
      const double yv = P == 0 ? y_cur[s] : ybar[s];
      double* o = red + P * kRowPer;
      const double es = s < m1 ? kx - qs : max0_ref(qs - kx);
      o[kPrS] += es * es;
      const double kxo = kx / r;
      const double eo = s < m1 ? kxo - qo : max0_ref(qo - kxo);
      o[kPrO] += eo * eo;
      o[kQyS] += qs * yv;
      o[kQyO] += qo * (yv * r);
      const double dy = yv - ys0;
      o[kDy2] += dy * dy;
    }
    if (!isfinite(y_cur[s])) red[2 * kRowPer] += 1.0;
  }
};

// Column side (kkt.cpp:78-103): lambda = proj(c - K'y), dual residual, bound
// term, c'x for both points and both spaces; dx for the primal weight
// (solver.cpp:433-436); finite test of x (solver.cpp:391). Two gathered
// operands: K^T [y_cur, ybar] from one pass over the matrix.
struct OpCheckCol {
  static constexpr int kRhs = 2, kRed = kColRed;
  static constexpr bool kMax = false;
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
  __device__ void map(int32_t i, double v, double (&p)[2]) const {
    p[0] = v * y_cur[i];
    p[1] = v * ybar[i];
  }
  __device__ void finish(int32_t s, const double (&a)[2], double* red) const {
    const double cS = c_s[s], lS = l_s[s], uS = u_s[s];
    const double cO = c_o[s], lO = l_o[s], uO = u_o[s], f = cs[s], x0 = x_start[s];
    const int cls = bound_class(lO, uO);
#pragma unroll
    for (int P = 0; P < 2; ++P) {
      const double kty = a[P];
      const double xv = P == 0 ? x_cur[s] : xbar[s];
      double* o = red + P * kColPer;
      const double rS = cS - kty;
      const double lamS = project_reduced(rS, cls);
      const double dS = rS - lamS;
      o[kDuS] += dS * dS;
      if (lamS > 0.0) o[kBdS] += lS * lamS;
      else if (lamS < 0.0) o[kBdS] += uS * lamS;
      const double rO = cO - kty / f;
      const double lamO = project_reduced(rO, cls);
      const double dO = rO - lamO;
      o[kDuO] += dO * dO;
      if (lamO > 0.0) o[kBdO] += lO * lamO;
      else if (lamO < 0.0) o[kBdO] += uO * lamO;
      o[kCxS] += cS * xv;
      o[kCxO] += cO * (xv * f);
      const double dx = xv - x0;
      o[kDx2] += dx * dx;
    }
    if (!isfinite(x_cur[s])) red[2 * kColPer] += 1.0;
  }
};

// DeriveLambda (kkt.cpp:127-141) for the returned y, original space.
struct OpLambda {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  const double* y_s;  // scaled dual
  const double* c_o;
  const double* l_o;
  const double* u_o;
  const double* cs;
  double* lam;
  __device__ void map(int32_t i, double v, double (&p)[1]) const { p[0] = v * y_s[i]; }
  __device__ void finish(int32_t s, const double (&a)[1], double*) const {
    lam[s] = project_reduced(c_o[s] - a[0] / cs[s], bound_class(l_o[s], u_o[s]));
  }
};

// PrimalStep / DualStep unit exports (solver.cpp:112-154) on an unscaled K.
struct OpUnitPrimal {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  const double* y;
  const double* x;
  const double* c;
  const double* l;
  const double* u;
  double step;  // eta / omega
  double* out;
  __device__ void map(int32_t i, double v, double (&p)[1]) const { p[0] = v * y[i]; }
  __device__ void finish(int32_t s, const double (&a)[1], double*) const {
    out[s] = clamp_ref(x[s] - step * (c[s] - a[0]), l[s], u[s]);
  }
};

struct OpUnitDual {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = false;
  const double* ext;  // 2 x_new - x_old
  const double* y;
  const double* q;
  int32_t m1;
  double step;  // eta * omega
  double* out;
  __device__ void map(int32_t j, double v, double (&p)[1]) const { p[0] = v * ext[j]; }
  __device__ void finish(int32_t s, const double (&a)[1], double*) const {
    const double v = y[s] + step * (q[s] - a[0]);
    out[s] = s < m1 ? v : max0_ref(v);
  }
};

}  // namespace pdhg
