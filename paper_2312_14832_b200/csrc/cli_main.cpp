// rpdlp-b200: the reference's command line tool (proj/tools/rpdlp_main.cpp:
// solve / bench / gen) over the C++ drop-in, with a small built-in option
// parser instead of CLI11 (absent here). Exit codes as the reference: 0 ok,
// 2 limit reached, 3 input error, 4 numerical failure; 1 for a usage error.
//
//   rpdlp-b200 solve FILE [--eps E] [--time-limit S] [--iter-limit N] [--log-every N]
//              [--check-every N] [--seed S] [--ruiz-iters N] [--pc-alpha A] [--out F]
//              [--no-scaling] [--no-restarts] [--adaptive-step] [--strict-mps]
//   rpdlp-b200 bench DIR [--eps E] [--time-limit S] [--iter-limit N] [--seed S] [--delta D]
//              [--report F] [--csv F] [--no-scaling] [--redact-timing]
//   rpdlp-b200 gen pagerank --nodes N [--damping D] [--attachment A] [--seed S] --out F
//   rpdlp-b200 gen random --rows M --cols N [--density D] [--seed S] --out F
//   rpdlp-b200 gen transport --sources S --sinks T [--seed S] --out F
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "rpdlp/bench.hpp"
#include "rpdlp/instance_gen.hpp"
#include "rpdlp/mps.hpp"
#include "rpdlp/solver.hpp"

namespace {

constexpr int kOk = 0, kUsage = 1, kLimit = 2, kInput = 3, kNumerical = 4;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Options of one subcommand: "--name" -> setter taking the value (flags take none).
class Options {
 public:
  void Value(const std::string& name, std::function<void(const std::string&)> set) { values_[name] = std::move(set); }
  void Flag(const std::string& name, bool* on) { flags_[name] = on; }
  void Required(const std::string& name) { required_.push_back(name); }
  // Parses argv[i..]; non-option words go to `positional`.
  void Parse(int argc, char** argv, int i, std::vector<std::string>* positional) {
    std::map<std::string, bool> seen;
    for (; i < argc; ++i) {
      const std::string a = argv[i];
      if (a.rfind("--", 0) != 0) {
        positional->push_back(a);
        continue;
      }
      if (auto f = flags_.find(a); f != flags_.end()) {
        *f->second = true;
      } else if (auto v = values_.find(a); v != values_.end()) {
        if (i + 1 >= argc) throw UsageError(a + " needs a value");
        try {
          v->second(argv[++i]);
        } catch (const std::logic_error&) {  // std::sto* failures
          throw UsageError("bad value for " + a + ": " + argv[i]);
        }
      } else {
        throw UsageError("unknown option " + a);
      }
      seen[a] = true;
    }
    for (const std::string& r : required_)
      if (!seen[r]) throw UsageError(r + " is required");
  }

 private:
  std::map<std::string, std::function<void(const std::string&)>> values_;
  std::map<std::string, bool*> flags_;
  std::vector<std::string> required_;
};

template <class T>
std::function<void(const std::string&)> Into(T* dst) {
  return [dst](const std::string& s) {
    if constexpr (std::is_same_v<T, std::string>) *dst = s;
    else if constexpr (std::is_floating_point_v<T>) *dst = std::stod(s);
    else if constexpr (std::is_unsigned_v<T>) *dst = static_cast<T>(std::stoull(s));
    else *dst = static_cast<T>(std::stoll(s));
  };
}

int Solve(int argc, char** argv) {
  rpdlp::SolverParams prm;
  std::string out;
  bool no_scaling = false, no_restarts = false, adaptive = false, strict = false;
  Options o;
  o.Value("--eps", Into(&prm.eps));
  o.Value("--time-limit", Into(&prm.time_limit));
  o.Value("--iter-limit", Into(&prm.iter_limit));
  o.Value("--log-every", Into(&prm.log_every));
  o.Value("--check-every", Into(&prm.check_every));
  o.Value("--seed", Into(&prm.seed));
  o.Value("--ruiz-iters", Into(&prm.scaling.ruiz_iters));
  o.Value("--pc-alpha", Into(&prm.scaling.pc_alpha));
  o.Value("--out", Into(&out));
  o.Flag("--no-scaling", &no_scaling);
  o.Flag("--no-restarts", &no_restarts);
  o.Flag("--adaptive-step", &adaptive);
  o.Flag("--strict-mps", &strict);
  rpdlp::DeviceOptions where;
  o.Value("--device", Into(&where.device));
  o.Value("--shards", Into(&where.shards));
  std::vector<std::string> pos;
  o.Parse(argc, argv, 2, &pos);
  if (pos.size() != 1) throw UsageError("solve takes one MPS file");
  rpdlp::MpsOptions mo;
  mo.fixed_format = strict;
  rpdlp::LpProblem problem;
  try {
    problem = rpdlp::ParseMpsFile(pos[0], mo);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kInput;
  }
  prm.scaling.enabled = !no_scaling;
  prm.restart_enabled = !no_restarts;
  prm.adaptive_step = adaptive;
  rpdlp::SolveResult r;
  try {
    r = rpdlp::Solve(problem, prm, nullptr, where);
  } catch (const rpdlp::NumericalFailure& e) {
    std::cerr << "numerical failure: " << e.what() << "\n";
    return kNumerical;
  }
  const double sign = problem.negated_objective ? -1.0 : 1.0;
  std::printf("status=%s objective=%.12e iterations=%lld restarts=%lld solve_seconds=%.3f\n",
              rpdlp::ToString(r.status).c_str(), sign * r.report.primal_obj, static_cast<long long>(r.iterations),
              static_cast<long long>(r.restarts), r.solve_seconds);
  if (!out.empty()) {
    std::ofstream f(out);
    if (!f) {
      std::cerr << "error: cannot write " << out << "\n";
      return kInput;
    }
    f << rpdlp::SolutionToJson(r, problem.negated_objective).dump(2) << "\n";
  }
  return r.status == rpdlp::SolveStatus::kOptimal ? kOk : kLimit;
}

int Bench(int argc, char** argv) {
  rpdlp::SolverParams prm;
  std::string report, csv;
  double delta = 10.0;
  bool no_scaling = false, redact = false;
  Options o;
  o.Value("--eps", Into(&prm.eps));
  o.Value("--time-limit", Into(&prm.time_limit));
  o.Value("--iter-limit", Into(&prm.iter_limit));
  o.Value("--seed", Into(&prm.seed));
  o.Value("--delta", Into(&delta));
  o.Value("--report", Into(&report));
  o.Value("--csv", Into(&csv));
  o.Flag("--no-scaling", &no_scaling);
  o.Flag("--redact-timing", &redact);
  rpdlp::SuiteOptions so;
  o.Value("--gpus", Into(&so.gpus));
  o.Value("--shards", Into(&so.shards));
  std::vector<std::string> pos;
  o.Parse(argc, argv, 2, &pos);
  if (pos.size() != 1) throw UsageError("bench takes one directory");
  prm.scaling.enabled = !no_scaling;
  rpdlp::SuiteSummary s;
  try {
    s = rpdlp::RunSuite(pos[0], prm, delta, so);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kInput;
  }
  for (const rpdlp::BenchRecord& r : s.records)
    std::printf("instance=%s status=%s solve_seconds=%.3f iterations=%lld\n", r.instance.c_str(), r.status.c_str(),
                r.solve_seconds, static_cast<long long>(r.iterations));
  std::printf("solved=%d/%zu sgm10=%.4f\n", s.solved_count, s.records.size(), s.sgm10);
  try {
    if (!report.empty()) rpdlp::WriteSummaryJson(s, report, redact);
    if (!csv.empty()) rpdlp::WriteSummaryCsv(s, csv);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kInput;
  }
  return kOk;
}

int Gen(int argc, char** argv) {
  if (argc < 3) throw UsageError("gen needs a kind: pagerank | random | transport");
  const std::string kind = argv[2];
  std::string out;
  Options o;
  o.Value("--out", Into(&out));
  o.Required("--out");
  std::vector<std::string> pos;
  rpdlp::LpProblem p;
  if (kind == "pagerank") {
    rpdlp::PagerankConfig cfg;
    o.Value("--nodes", Into(&cfg.n_nodes));
    o.Value("--damping", Into(&cfg.damping));
    o.Value("--attachment", Into(&cfg.attachment));
    o.Value("--seed", Into(&cfg.seed));
    o.Required("--nodes");
    o.Parse(argc, argv, 3, &pos);
    p = rpdlp::GenPagerank(cfg);
  } else if (kind == "random") {
    rpdlp::Index rows = 0, cols = 0;
    double density = 0.5;
    std::uint64_t seed = 0;
    o.Value("--rows", Into(&rows));
    o.Value("--cols", Into(&cols));
    o.Value("--density", Into(&density));
    o.Value("--seed", Into(&seed));
    o.Required("--rows");
    o.Required("--cols");
    o.Parse(argc, argv, 3, &pos);
    p = rpdlp::GenRandomLp(rows, cols, density, seed);
  } else if (kind == "transport") {
    rpdlp::Index sources = 0, sinks = 0;
    std::uint64_t seed = 1;
    o.Value("--sources", Into(&sources));
    o.Value("--sinks", Into(&sinks));
    o.Value("--seed", Into(&seed));
    o.Required("--sources");
    o.Required("--sinks");
    o.Parse(argc, argv, 3, &pos);
    p = rpdlp::GenTransport(sources, sinks, seed);
  } else {
    throw UsageError("unknown instance kind " + kind);
  }
  if (!pos.empty()) throw UsageError("unexpected argument " + pos[0]);
  rpdlp::WriteMpsFile(p, out);
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string cmd = argc > 1 ? argv[1] : "";
  try {
    if (cmd == "solve") return Solve(argc, argv);
    if (cmd == "bench") return Bench(argc, argv);
    if (cmd == "gen") return Gen(argc, argv);
    throw UsageError(cmd.empty() ? "a subcommand is required: solve | bench | gen" : "unknown subcommand " + cmd);
  } catch (const UsageError& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::exception& e) {  // rpdlp_main.cpp:212-215
    std::cerr << "error: " << e.what() << "\n";
    return kInput;
  }
}
