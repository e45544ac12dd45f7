// Drop-in ScalingConfig (reference proj/core/include/rpdlp/scaling.hpp:40-44).
// Ruiz / Pock-Chambolle / ApplyScaling run on the device inside Solve.
#ifndef RPDLP_B200_SCALING_HPP_
#define RPDLP_B200_SCALING_HPP_

namespace rpdlp {

struct ScalingConfig {
  bool enabled = true;
  int ruiz_iters = 10;
  double pc_alpha = 1.0;
};

}  // namespace rpdlp

#endif  // RPDLP_B200_SCALING_HPP_
