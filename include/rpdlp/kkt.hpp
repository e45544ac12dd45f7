// Drop-in KKT types and helpers (reference proj/core/include/rpdlp/kkt.hpp:25-77).
#ifndef RPDLP_B200_KKT_HPP_
#define RPDLP_B200_KKT_HPP_

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

}  // namespace rpdlp

#endif  // RPDLP_B200_KKT_HPP_
