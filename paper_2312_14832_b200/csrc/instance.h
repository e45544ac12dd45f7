// Host-owned LP instance (generators, MPS reader): the arrays a pdhg_lp view
// points into (include/pdhg.h). Internal to libpdhg_b200.so.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

struct pdhg_instance {
  int64_t n = 0;
  int64_t a_rows = 0, g_rows = 0;
  std::vector<int64_t> a_ptr{0}, a_idx, g_ptr{0}, g_idx;
  std::vector<double> a_val, g_val, c, b, h, l, u, witness;
  double offset = 0.0;
  int32_t negated = 0;
  std::string name;
};
