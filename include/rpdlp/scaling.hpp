// Drop-in scaling API (reference proj/core/include/rpdlp/scaling.hpp:30-59).
// RuizEquilibrate / PockChambolleScale / ComputeScaling run on the device
// (pdhg_compute_scaling, $PDHG_DEVICE); ApplyScaling and the ScalingInfo
// helpers are host code with the reference's operations and rounding order.
#ifndef RPDLP_B200_SCALING_HPP_
#define RPDLP_B200_SCALING_HPP_

#include <span>
#include <vector>

#include "rpdlp/lp_problem.hpp"

namespace rpdlp {

struct ScalingInfo {
  std::vector<double> row_scale;  // length m1 + m2
  std::vector<double> col_scale;  // length n

  static ScalingInfo Identity(Index n_rows, Index n_cols);
  ScalingInfo Composed(const ScalingInfo& other) const;  // entrywise product
  void UnscaleIterate(std::span<double> x, std::span<double> y) const;
};

struct ScalingConfig {
  bool enabled = true;
  int ruiz_iters = 10;
  double pc_alpha = 1.0;
};

ScalingInfo RuizEquilibrate(const SparseMatrix& k, int iters);
ScalingInfo PockChambolleScale(const SparseMatrix& k, double alpha);
ScalingInfo ComputeScaling(const SparseMatrix& k, const ScalingConfig& config);
LpProblem ApplyScaling(const LpProblem& problem, const ScalingInfo& info);

}  // namespace rpdlp

#endif  // RPDLP_B200_SCALING_HPP_
