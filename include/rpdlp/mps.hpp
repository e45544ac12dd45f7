// Drop-in MPS reader/writer (reference proj/core/include/rpdlp/mps.hpp:26-56),
// backed by pdhg_mps_* in libpdhg_b200 (same normalisations, exceptions and
// messages; see csrc/mps.cpp).
#ifndef RPDLP_B200_MPS_HPP_
#define RPDLP_B200_MPS_HPP_

#include <iosfwd>
#include <stdexcept>
#include <string>

#include "rpdlp/lp_problem.hpp"

namespace rpdlp {

class MpsParseError : public std::runtime_error {
 public:
  MpsParseError(int line, const std::string& message)
      : std::runtime_error("mps parse error at line " + std::to_string(line) + ": " + message), line_(line) {}
  int line() const { return line_; }

 private:
  int line_;
};

struct MpsOptions {
  bool fixed_format = false;
};

LpProblem ParseMps(std::istream& in, const MpsOptions& options = {});
LpProblem ParseMpsString(const std::string& text, const MpsOptions& = {});
LpProblem ParseMpsFile(const std::string& path, const MpsOptions& = {});

void WriteMps(const LpProblem& problem, std::ostream& out);
void WriteMpsFile(const LpProblem& problem, const std::string& path);

}  // namespace rpdlp

#endif  // RPDLP_B200_MPS_HPP_
