// Drop-in check: reference-style C++ caller code compiled against
// include/rpdlp/*.hpp and linked to libpdhg_b200.so (no reference code).
// Cases follow the reference's own unit tests (test_solver.cpp, test_kkt.cpp)
// and acceptance criteria C1/C5 shapes. Exit code = number of failures.
#include <cmath>
#include <fstream>
#include <cstdlib>
#include <random>
#include <cstdio>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include <sstream>

#include "rpdlp/bench.hpp"
#include "rpdlp/instance_gen.hpp"
#include "rpdlp/kkt.hpp"
#include "rpdlp/mps.hpp"
#include "rpdlp/scaling.hpp"
#include "rpdlp/solver.hpp"

using namespace rpdlp;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (cond) {                                                          \
      ++g_pass;                                                          \
    } else {                                                             \
      ++g_fail;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                    \
  } while (0)

static bool Near(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(1.0, std::abs(b)); }

static LpProblem TinyLp() {
  LpProblem p;
  p.a = SparseMatrix::FromTriplets(0, 1, {});
  p.g = SparseMatrix::FromTriplets(1, 1, {{0, 0, 1.0}});
  p.c = {1.0};
  p.h = {1.0};
  p.l = {0.0};
  p.u = {kInf};
  return p;
}

int main() {
  {  // test_solver.cpp:198-208
    SolverParams prm;
    prm.eps = 1e-8;
    SolveResult r = Solve(TinyLp(), prm);
    CHECK(r.status == SolveStatus::kOptimal);
    CHECK(Near(r.x[0], 1.0, 1e-6) && Near(r.y[0], 1.0, 1e-6));
    CHECK(r.report.rel_primal <= 1e-8 && r.report.rel_dual <= 1e-8 && r.report.rel_gap <= 1e-8);
  }
  {  // operator norms (test_solver.cpp:41-57)
    CHECK(Near(EstimateOpNorm(SparseMatrix::FromTriplets(1, 1, {{0, 0, 3.0}}), 50, 1), 3.0, 1e-12));
    const double est = EstimateOpNorm(SparseMatrix::FromTriplets(3, 3, {{0, 0, 1.0}, {1, 1, 2.0}, {2, 2, 5.0}}), 200, 1);
    CHECK(est > 4.95 && est <= 5.0 + 1e-12);
    CHECK(EstimateOpNorm(SparseMatrix::FromTriplets(2, 3, {}), 20, 1) == 0.0);
  }
  {  // PrimalStep / DualStep hand examples (test_solver.cpp:65-112)
    LpProblem p;
    p.a = SparseMatrix::FromTriplets(0, 1, {});
    p.g = SparseMatrix::FromTriplets(1, 1, {{0, 0, 1.0}});
    p.c = {1.0};
    p.h = {0.0};
    p.l = {0.0};
    p.u = {1.0};
    CHECK(PrimalStep(p, std::vector<double>{0.2}, std::vector<double>{0.5}, 0.5, 1.0)[0] == 0.0);
    CHECK(Near(PrimalStep(p, std::vector<double>{0.2}, std::vector<double>{0.5}, 0.5, 2.0)[0], 0.075, 1e-15));
    CHECK(PrimalStep(p, std::vector<double>{0.9}, std::vector<double>{5.0}, 0.5, 1.0)[0] == 1.0);
    LpProblem d;
    d.a = SparseMatrix::FromTriplets(1, 1, {{0, 0, 1.0}});
    d.g = SparseMatrix::FromTriplets(1, 1, {{0, 0, 1.0}});
    d.c = {0.0};
    d.b = {2.0};
    d.h = {2.0};
    d.l = {0.0};
    d.u = {kInf};
    auto y = DualStep(d, std::vector<double>{1.0}, std::vector<double>{0.5}, std::vector<double>{0.1, 0.1}, 0.5, 1.0);
    CHECK(Near(y[0], 0.35, 1e-15) && Near(y[1], 0.35, 1e-15));
    auto y2 = DualStep(d, std::vector<double>{3.0}, std::vector<double>{3.0}, std::vector<double>{0.1, 0.1}, 0.5, 1.0);
    CHECK(Near(y2[0], -0.4, 1e-15) && y2[1] == 0.0);
  }
  {  // restart truth table (test_solver.cpp:155-183)
    SolverParams prm;
    const double inf = std::numeric_limits<double>::infinity();
    CHECK(ShouldRestart(prm, 1, 100, 0.10, 1.0, 0.05));
    CHECK(ShouldRestart(prm, 1, 100, 0.50, 1.0, 0.40));
    CHECK(!ShouldRestart(prm, 1, 100, 0.50, 1.0, 0.60));
    CHECK(ShouldRestart(prm, 36, 100, 0.90, 1.0, inf));
    CHECK(!ShouldRestart(prm, 35, 100, 0.90, 1.0, inf));
    CHECK(Near(UpdatePrimalWeight(1.0, 1.0, 4.0), 2.0, 1e-15));
    CHECK(Near(KktError(3.0, 4.0, 0.0, 1.0), 5.0, 1e-15));
  }
  {  // limits (test_solver.cpp:251-263)
    SolverParams prm;
    prm.eps = 1e-16;
    prm.iter_limit = 10;
    SolveResult r = Solve(GenRandomLp(5, 5, 0.6, 7), prm);
    CHECK(r.status == SolveStatus::kIterLimit && r.iterations <= 10);
    prm.iter_limit = std::numeric_limits<Index>::max();
    prm.time_limit = 0.0;
    CHECK(Solve(GenRandomLp(5, 5, 0.6, 7), prm).status == SolveStatus::kTimeLimit);
  }
  {  // errors map back to the reference's exception types
    LpProblem p = TinyLp();
    p.l = {2.0};
    p.u = {1.0};
    bool threw = false;
    try {
      Solve(p, SolverParams{});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    SolverParams bad;
    bad.check_every = 0;
    threw = false;
    try {
      Solve(TinyLp(), bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // observer (test_solver.cpp:277-292) and its exceptions
    SolverParams prm;
    prm.eps = 1e-6;
    Index last = -1, seen = 0;
    bool order = true;
    SolveResult r = Solve(GenPagerank({200, 0.85, 3, 4}), prm, [&](const EvalInfo& e) {
      if (e.iteration < last) order = false;
      last = e.iteration;
      seen += e.restarted;
    });
    CHECK(r.status == SolveStatus::kOptimal && order && seen == r.restarts);
    bool threw = false;
    try {
      Solve(GenPagerank({200, 0.85, 3, 4}), prm, [](const EvalInfo&) { throw std::runtime_error("stop"); });
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()) == "stop";
    }
    CHECK(threw);
  }
  {  // acceptance C5 shape: PageRank n in {100, 1000, 10000} at 1e-6
    for (Index n : {100, 1000, 10000}) {
      SolverParams prm;
      prm.eps = 1e-6;
      SolveResult r = Solve(GenPagerank({n, 0.85, 3, 2026}), prm);
      const double s = std::accumulate(r.x.begin(), r.x.end(), 0.0);
      CHECK(r.status == SolveStatus::kOptimal);
      CHECK(std::abs(s - 1.0) <= 1e-4);
      double mn = 0.0;
      for (double v : r.x) mn = std::min(mn, v);
      CHECK(mn >= 0.0);
    }
  }
  {  // determinism (test_solver.cpp:265-275)
    SolverParams prm;
    prm.eps = 1e-8;
    LpProblem p = GenRandomLp(6, 8, 0.5, 55);
    SolveResult a = Solve(p, prm), b = Solve(p, prm);
    CHECK(a.iterations == b.iterations && a.x == b.x && a.y == b.y);
  }
  {  // MPS ingestion (mps.hpp / test_mps.cpp): parse, errors, write round trip, solve
    const std::string text =
        "NAME T\nROWS\n N obj\n E e1\n L l1\nCOLUMNS\n x obj 1 e1 1\n x l1 1\n y obj 2 e1 1\n"
        "RHS\n RHS e1 2 l1 1.5\nBOUNDS\n UP B y 3\nENDATA\n";
    LpProblem p = ParseMpsString(text);
    CHECK(p.name == "T" && p.num_vars() == 2 && p.num_eq_rows() == 1 && p.num_ineq_rows() == 1);
    CHECK(p.h[0] == -1.5 && p.u[1] == 3.0);
    bool threw = false;
    try {
      ParseMpsString("NAME\nROWS\n N o\n Q r\n");
    } catch (const MpsParseError& e) {
      threw = e.line() == 4 && std::string(e.what()) == "mps parse error at line 4: unknown row type 'Q'";
    }
    CHECK(threw);
    std::ostringstream os;
    WriteMps(p, os);
    LpProblem q = ParseMpsString(os.str());
    CHECK(q.c == p.c && q.b == p.b && q.h == p.h && q.l == p.l && q.u == p.u);
    SolverParams prm;
    prm.eps = 1e-8;
    SolveResult r = Solve(q, prm);
    CHECK(r.status == SolveStatus::kOptimal && Near(r.report.primal_obj, 2.5, 1e-6));  // x = 1.5, y = 0.5
  }
  {  // the new SURVEY §8d shapes through the drop-in generators
    SolverParams prm;
    prm.eps = 1e-4;
    SolveResult r = Solve(GenMcf(40, 200, 3, 1), prm);
    CHECK(r.status == SolveStatus::kOptimal);
    SolveResult s = Solve(GenStaircase(4, 20, 25, 6, 2, 10, 1), prm);
    CHECK(s.status == SolveStatus::kOptimal);
  }
  {  // scaling + residual API (test_scaling.cpp:27-180, test_kkt.cpp:65-101)
    const SparseMatrix one = SparseMatrix::FromTriplets(1, 1, {{0, 0, 100.0}});
    CHECK(Near(RuizEquilibrate(one, 10).row_scale[0], 0.1, 1e-15));
    LpProblem p = GenRandomLp(20, 30, 0.3, 9);
    const SparseMatrix& k = p.g;
    ScalingInfo info = ComputeScaling(k, ScalingConfig{});
    LpProblem s = ApplyScaling(p, info);
    SolverParams prm;
    prm.eps = 1e-8;
    prm.scaling.enabled = false;
    SolveResult rs = Solve(s, prm);
    info.UnscaleIterate(rs.x, rs.y);
    SolveResult ro = Solve(p, prm);
    CHECK(std::abs(rs.report.primal_obj - ro.report.primal_obj) <= 1e-6 * (1.0 + std::abs(ro.report.primal_obj)));
    const ResidualReport r = ComputeResiduals(p, Iterate{ro.x, ro.y});
    CHECK(r.rel_primal <= 1e-8 && r.rel_dual <= 1e-8 && r.rel_gap <= 1e-8);
    ResidualEvaluator ev(p);
    CHECK(Near(ev.KktOmega(ro.x, ro.y, 1.0), KktError(r.primal_res, r.dual_res, r.gap_abs, 1.0), 1e-12));
    const std::vector<double> lam = DeriveLambda(p, ro.y);
    CHECK(lam.size() == ro.lambda.size());
    double dl = 0.0;
    for (size_t j = 0; j < lam.size(); ++j) dl = std::max(dl, std::abs(lam[j] - ro.lambda[j]));
    CHECK(dl <= 1e-12);
  }
  {  // GenPagerankGraph / BuildPagerankLp / ReadEdgeList (instance_gen.cpp:27-141)
    PagerankConfig cfg;
    cfg.n_nodes = 2000;
    cfg.attachment = 4;
    cfg.seed = 7;
    const EdgeList e = GenPagerankGraph(cfg);
    CHECK(e.size() == static_cast<size_t>(5 + (2000 - 5) * 4));
    const LpProblem a = BuildPagerankLp(e, cfg.n_nodes, cfg.damping), b = GenPagerank(cfg);
    CHECK(a.g == b.g && a.a == b.a && a.h == b.h && a.name == "pagerank");
    const std::string path = "/tmp/rpdlp_b200_edges_test.txt";
    {
      std::FILE* f = std::fopen(path.c_str(), "w");
      std::fputs("# comment\n\n10 20\n  20 30\n30 10\n", f);
      std::fclose(f);
    }
    Index n = 0;
    const EdgeList r = ReadEdgeList(path, &n);
    CHECK(n == 3 && r.size() == 3 && r[0] == std::make_pair(Index(0), Index(1)) && r[2] == std::make_pair(Index(2), Index(0)));
    bool threw = false;
    try {
      BuildPagerankLp({{0, 9}}, 3, 0.85);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    std::remove(path.c_str());
  }
  {  // suite harness (test_bench.cpp: SGM hand values, run_suite, byte-identical redacted reports)
    CHECK(Near(Sgm({10.0, 40.0}, 10.0, 3600.0, {true, true}), std::sqrt(1000.0) - 10.0, 1e-12));
    CHECK(Near(Sgm({1.0, 2.0}, 10.0, 100.0, {true, false}), std::sqrt(11.0 * 110.0) - 10.0, 1e-12));
    bool threw = false;
    try {
      Sgm({}, 10.0, 3600.0, {});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    const std::string dir = "/tmp/rpdlp_b200_suite_test";
    std::system(("rm -rf " + dir + " && mkdir -p " + dir).c_str());
    WriteMpsFile(GenRandomLp(6, 7, 0.5, 1), dir + "/a.mps");
    WriteMpsFile(GenRandomLp(6, 7, 0.5, 2), dir + "/b.mps");
    {
      std::FILE* f = std::fopen((dir + "/broken.mps").c_str(), "w");
      std::fputs("ROWS\n N OBJ\nCOLUMNS\n", f);
      std::fclose(f);
    }
    SolverParams prm;
    prm.eps = 1e-6;
    const SuiteSummary s1 = RunSuite(dir, prm), s2 = RunSuite(dir, prm);
    CHECK(s1.records.size() == 3 && s1.solved_count == 2 && s1.records[2].status == "Error");
    CHECK(s1.records[0].instance == "a.mps" && s1.records[0].iterations > 0 && s1.sgm10 > 0.0);
    CHECK(SummaryToJson(s1, true).dump(2) == SummaryToJson(s2, true).dump(2));
    const auto j = SummaryToJson(s1);
    CHECK(j.begin().key() == "tolerance" && j["records"][0]["residuals"].size() == 8 && j["solved_count"] == 2);
    WriteSummaryCsv(s1, dir + "/r.csv");
    std::ifstream csv(dir + "/r.csv");
    std::string header;
    std::getline(csv, header);
    CHECK(header == "instance,status,solve_seconds,parse_seconds,scaling_seconds,iterations,restarts,rel_primal,"
                    "rel_dual,rel_gap,primal_obj");
    const SolveResult r = Solve(GenRandomLp(6, 7, 0.5, 1), prm);
    const auto sol = SolutionToJson(r, true);
    CHECK(sol["status"] == "Optimal" && sol["primal_objective"].get<double>() == -r.report.primal_obj &&
          sol["x"].size() == r.x.size());
    std::system(("rm -rf " + dir).c_str());
  }
  {  // SparseMatrix SpMV members (test_sparse_matrix.cpp:80-101): device result vs the serial row sums
    const LpProblem p = GenRandomLp(40, 30, 0.3, 11);
    const SparseMatrix& k = p.g;
    std::vector<double> x(k.cols()), yr(k.rows());
    for (size_t j = 0; j < x.size(); ++j) x[j] = std::sin(1.0 + j);
    for (size_t i = 0; i < yr.size(); ++i) yr[i] = std::cos(2.0 + i);
    std::vector<double> y(k.rows()), want(k.rows(), 0.0);
    k.Multiply(x, y);
    for (Index r = 0; r < k.rows(); ++r) {
      double acc = 0.0;
      for (Index q = k.row_ptr()[r]; q < k.row_ptr()[r + 1]; ++q) acc += k.csr_values()[q] * x[k.col_idx()[q]];
      want[r] = acc;
    }
    CHECK(y == want);  // storage-order sums: bit-identical
    std::vector<double> z(k.cols()), wantz(k.cols(), 0.0);
    k.MultiplyTranspose(yr, z);
    for (Index c = 0; c < k.cols(); ++c) {
      double acc = 0.0;
      for (Index q = k.col_ptr()[c]; q < k.col_ptr()[c + 1]; ++q) acc += k.csc_values()[q] * yr[k.row_idx()[q]];
      wantz[c] = acc;
    }
    CHECK(z == wantz);
    std::vector<double> acc(k.rows(), 1.0);
    k.MultiplyAdd(-2.0, x, acc);
    bool ok = true;
    for (Index r = 0; r < k.rows(); ++r) ok = ok && acc[r] == 1.0 + -2.0 * want[r];
    CHECK(ok);
    // norms / power sums / Scaled (sparse_matrix.cpp:166-222) against serial loops
    std::vector<double> rinf(k.rows(), 0.0), cinf(k.cols(), 0.0), rp1(k.rows(), 0.0), cp2(k.cols(), 0.0);
    for (Index r = 0; r < k.rows(); ++r)
      for (Index q = k.row_ptr()[r]; q < k.row_ptr()[r + 1]; ++q) {
        rinf[r] = std::max(rinf[r], std::abs(k.csr_values()[q]));
        rp1[r] += std::abs(k.csr_values()[q]);
      }
    for (Index c = 0; c < k.cols(); ++c)
      for (Index q = k.col_ptr()[c]; q < k.col_ptr()[c + 1]; ++q) {
        cinf[c] = std::max(cinf[c], std::abs(k.csc_values()[q]));
        cp2[c] += k.csc_values()[q] * k.csc_values()[q];
      }
    CHECK(k.RowInfNorms() == rinf && k.ColInfNorms() == cinf && k.RowPowerSums(1.0) == rp1 &&
          k.ColPowerSums(2.0) == cp2);
    const SparseMatrix s = k.Scaled(yr, x);
    bool sok = s.row_ptr() == k.row_ptr() && s.col_idx() == k.col_idx();
    for (Index r = 0; r < k.rows(); ++r)
      for (Index q = k.row_ptr()[r]; q < k.row_ptr()[r + 1]; ++q)
        sok = sok && s.csr_values()[q] == yr[r] * k.csr_values()[q] * x[k.col_idx()[q]];
    for (Index c = 0; c < k.cols(); ++c)
      for (Index q = k.col_ptr()[c]; q < k.col_ptr()[c + 1]; ++q)
        sok = sok && s.csc_values()[q] == yr[k.row_idx()[q]] * k.csc_values()[q] * x[c];
    CHECK(sok);
    bool threw = false;
    try {
      k.Multiply(yr, y);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // ChooseRestartCandidate (solver.cpp:170-176, test_solver.cpp restart tests): strict < picks current
    LpProblem p = GenRandomLp(10, 12, 0.4, 4);
    SolverParams prm;
    prm.eps = 1e-8;
    SolveResult r = Solve(p, prm);
    const Iterate good{r.x, r.y};
    const Iterate zero{std::vector<double>(r.x.size(), 0.0), std::vector<double>(r.y.size(), 0.0)};
    CHECK(ChooseRestartCandidate(p, good, zero, 1.0) == good);
    CHECK(ChooseRestartCandidate(p, zero, good, 1.0) == good);
    const Iterate same = good;
    CHECK(ChooseRestartCandidate(p, good, same, 1.0) == same);  // tie -> average
  }
  {  // >= 2^20 triplets take the device assembly (pdhg_csr_from_triplets): same matrix as the host path
    std::mt19937_64 g(5);
    std::vector<Triplet> t(1200000);
    for (Triplet& e : t) {
      e.row = static_cast<Index>(g() % 5000);
      e.col = static_cast<Index>(g() % 4000);
      e.value = static_cast<double>(static_cast<int>(g() % 33) - 16) / 8.0;  // dyadic: duplicate sums exact
    }
    setenv("PDHG_DEVICE_ASSEMBLY", "0", 1);
    const SparseMatrix h = SparseMatrix::FromTriplets(5000, 4000, t);
    unsetenv("PDHG_DEVICE_ASSEMBLY");
    const SparseMatrix d = SparseMatrix::FromTriplets(5000, 4000, t);
    CHECK(h.nnz() > 1000000 && h == d);
    t.push_back({5000, 0, 1.0});
    bool threw = false;
    try {
      SparseMatrix::FromTriplets(5000, 4000, t);
    } catch (const std::out_of_range&) {
      threw = true;
    }
    CHECK(threw);
  }
  std::printf("drop_in_test: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
