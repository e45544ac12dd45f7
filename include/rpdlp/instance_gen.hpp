// Drop-in instance generators (reference proj/core/include/rpdlp/instance_gen.hpp:27-59),
// bit-identical per seed; backed by pdhg_gen_* in libpdhg_b200.
#ifndef RPDLP_B200_INSTANCE_GEN_HPP_
#define RPDLP_B200_INSTANCE_GEN_HPP_

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "rpdlp/lp_problem.hpp"

namespace rpdlp {

struct PagerankConfig {
  Index n_nodes = 0;
  double damping = 0.85;
  Index attachment = 3;
  std::uint64_t seed = 0;
};

// Directed edge list, src -> dst (instance_gen.hpp:34-49).
using EdgeList = std::vector<std::pair<Index, Index>>;
// Preferential-attachment digraph, deterministic per seed (bit-identical
// with the reference's draw).
EdgeList GenPagerankGraph(const PagerankConfig& cfg);
// "src dst" per line, '#' comment lines; ids compacted to 0..n-1 in order of
// first appearance. Throws std::runtime_error (cannot open / malformed line).
EdgeList ReadEdgeList(const std::string& path, Index* n_nodes);
// Feasibility LP of x = damping S x + (1 - damping)/n (see pdhg.h).
LpProblem BuildPagerankLp(const EdgeList& edges, Index n_nodes, double damping);
LpProblem GenPagerank(const PagerankConfig& cfg);
LpProblem GenRandomLp(Index m, Index n, double density, std::uint64_t seed, std::vector<double>* witness = nullptr);
// SURVEY §8d config 2 (not in the reference).
LpProblem GenTransport(Index sources, Index sinks, std::uint64_t seed);
// SURVEY §8d configs 3 (multicommodity flow) and 5 (block-angular staircase).
LpProblem GenMcf(Index nodes, Index arcs, Index commodities, std::uint64_t seed,
                 std::vector<double>* witness = nullptr);
LpProblem GenStaircase(Index stages, Index rows_per_stage, Index cols_per_stage, Index nnz_per_row,
                       Index linking_per_row, Index eq_rows_per_stage, std::uint64_t seed,
                       std::vector<double>* witness = nullptr);

}  // namespace rpdlp

#endif  // RPDLP_B200_INSTANCE_GEN_HPP_
