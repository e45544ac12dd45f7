// Drop-in instance generators (reference proj/core/include/rpdlp/instance_gen.hpp:27-59),
// bit-identical per seed; backed by pdhg_gen_* in libpdhg_b200.
#ifndef RPDLP_B200_INSTANCE_GEN_HPP_
#define RPDLP_B200_INSTANCE_GEN_HPP_

#include <cstdint>
#include <vector>

#include "rpdlp/lp_problem.hpp"

namespace rpdlp {

struct PagerankConfig {
  Index n_nodes = 0;
  double damping = 0.85;
  Index attachment = 3;
  std::uint64_t seed = 0;
};

LpProblem GenPagerank(const PagerankConfig& cfg);
LpProblem GenRandomLp(Index m, Index n, double density, std::uint64_t seed, std::vector<double>* witness = nullptr);
// SURVEY §8d config 2 (not in the reference).
LpProblem GenTransport(Index sources, Index sinks, std::uint64_t seed);

}  // namespace rpdlp

#endif  // RPDLP_B200_INSTANCE_GEN_HPP_
