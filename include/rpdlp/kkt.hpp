// Drop-in KKT types and helpers (reference proj/core/include/rpdlp/kkt.hpp:25-77).
#ifndef RPDLP_B200_KKT_HPP_
#define RPDLP_B200_KKT_HPP_

#include <span>
#include <vector>

#include "rpdlp/lp_problem.hpp"

namespace rpdlp {

struct Iterate {
  std::vector<double> x;
  std::vector<double> y;
  bool operator==(const Iterate& other) const = default;
};

struct ResidualReport {
  double primal_res = 0.0;
  double dual_res = 0.0;
  double gap_abs = 0.0;
  double primal_obj = 0.0;
  double dual_obj = 0.0;
  double rel_primal = 0.0;
  double rel_dual = 0.0;
  double rel_gap = 0.0;
};

bool CheckTermination(const ResidualReport& report, double eps);
double KktError(double primal_res, double dual_res, double gap, double omega);

// Device-backed (pdhg_residuals / pdhg_derive_lambda; $PDHG_DEVICE).
std::vector<double> DeriveLambda(const LpProblem& problem, std::span<const double> y);
ResidualReport ComputeResiduals(const LpProblem& problem, const Iterate& z);
double KktOmega(const LpProblem& problem, const Iterate& z, double omega);

// kkt.hpp:59-77 interface; each Evaluate is one device residual pass.
class ResidualEvaluator {
 public:
  explicit ResidualEvaluator(const LpProblem& problem);
  ResidualReport Evaluate(std::span<const double> x, std::span<const double> y) const;
  double KktOmega(std::span<const double> x, std::span<const double> y, double omega) const;
  double q_norm() const { return q_norm_; }
  double c_norm() const { return c_norm_; }

 private:
  const LpProblem& problem_;
  double q_norm_;
  double c_norm_;
};

}  // namespace rpdlp

#endif  // RPDLP_B200_KKT_HPP_
