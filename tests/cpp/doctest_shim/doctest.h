// Minimal doctest-compatible test runner -- test infrastructure only.
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// <doctest.h>, whose vendored copy is absent from the reference tree and not
// installable here. This header implements exactly the subset
// those files use, with doctest's semantics, so they compile UNCHANGED against
// include/rpdlp/*.hpp + libpdhg_b200.so (tests/cpp/Makefile):
//
//   TEST_CASE, SUBCASE (flat siblings: the test body re-runs once per leaf,
//   code outside subcases runs every pass), CHECK, CHECK_FALSE, REQUIRE,
//   CHECK_THROWS_AS, CHECK_THROWS_WITH_AS (exact what() match), CAPTURE,
//   FAIL, doctest::Approx with .epsilon() / .scale() (doctest's relative
//   comparison: |a-b| < eps * (scale + max(|a|, |b|)), default eps =
//   100 * FLT_EPSILON, scale 1).
//
// The runner prints a doctest-style summary ("[doctest] test cases: N | P
// passed | F failed") and exits with the number of failed test cases.
// Optional argv: -tc=<substring> filters test cases by name.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool eq(double other) const {
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
  }
  double value() const { return value_; }

  friend bool operator==(double a, const Approx& b) { return b.eq(a); }
  friend bool operator==(const Approx& a, double b) { return a.eq(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
  friend bool operator!=(const Approx& a, double b) { return !a.eq(b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.eq(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.eq(a); }
  friend bool operator<=(const Approx& a, double b) { return a.value_ < b || a.eq(b); }
  friend bool operator>=(const Approx& a, double b) { return a.value_ > b || a.eq(b); }
  friend bool operator<(double a, const Approx& b) { return a < b.value_ && !b.eq(a); }
  friend bool operator>(double a, const Approx& b) { return a > b.value_ && !b.eq(a); }
  friend bool operator<(const Approx& a, double b) { return a.value_ < b && !a.eq(b); }
  friend bool operator>(const Approx& a, double b) { return a.value_ > b && !a.eq(b); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace shim {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

// Thrown by REQUIRE / FAIL to leave the current test case.
struct Abort {};

struct State {
  const TestCase* current = nullptr;
  bool failed = false;
  long assertions = 0, failed_assertions = 0;
  // Flat SUBCASE traversal: leaves already run, and whether this pass
  // entered one.
  std::set<std::string> done;
  bool entered = false, pending = false;
  std::string subcase;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

inline void report_failure(const char* file, int line, const std::string& what) {
  State& s = state();
  s.failed = true;
  ++s.failed_assertions;
  std::printf("%s:%d: ERROR: %s\n", file, line, what.c_str());
  std::printf("  in TEST_CASE(\"%s\")%s%s\n", s.current ? s.current->name : "?",
              s.subcase.empty() ? "" : " SUBCASE ", s.subcase.c_str());
  for (const std::string& c : s.captures) std::printf("  logged: %s\n", c.c_str());
}

inline bool check(bool ok, const char* file, int line, const char* macro, const char* expr) {
  ++state().assertions;
  if (!ok) report_failure(file, line, std::string(macro) + "( " + expr + " ) is NOT correct!");
  return ok;
}

struct Subcase {
  std::string key;
  bool run = false;
  Subcase(const char* name, const char* file, int line) {
    State& s = state();
    key = std::string(file) + ":" + std::to_string(line) + ":" + name;
    if (!s.entered && s.done.count(key) == 0) {
      s.entered = true;
      s.done.insert(key);
      s.subcase = name;
      run = true;
    } else if (s.done.count(key) == 0) {
      s.pending = true;  // seen behind the one this pass runs
    }
  }
  explicit operator bool() const { return run; }
};

struct Capture {
  explicit Capture(std::string s) { state().captures.push_back(std::move(s)); }
  ~Capture() { state().captures.pop_back(); }
};

template <class T>
std::string to_text(const char* expr, const T& v) {
  std::ostringstream os;
  os << expr << " := " << v;
  return os.str();
}

inline int run_all(int argc, char** argv) {
  std::string filter;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
  }
  State& s = state();
  int total = 0, failed = 0, skipped = 0;
  for (const TestCase& tc : registry()) {
    if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) {
      ++skipped;
      continue;
    }
    ++total;
    s.current = &tc;
    s.failed = false;
    s.done.clear();
    // Re-run the body while a pass skipped a not-yet-run subcase.
    for (;;) {
      s.entered = s.pending = false;
      s.subcase.clear();
      s.captures.clear();
      try {
        tc.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        report_failure(tc.file, tc.line, std::string("TEST CASE THREW exception: ") + e.what());
      } catch (...) {
        report_failure(tc.file, tc.line, "TEST CASE THREW an unknown exception");
      }
      if (!s.pending) break;
    }
    if (s.failed) ++failed;
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", total, total - failed, failed,
              skipped);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed |\n", s.assertions,
              s.assertions - s.failed_assertions, s.failed_assertions);
  std::printf("[doctest] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
  return failed;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(p) DOCTEST_CAT(p, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                               \
  static void fn();                                                                         \
  static const ::doctest::shim::Registrar reg(name, __FILE__, __LINE__, &fn);               \
  static void fn()
#define DOCTEST_TEST_CASE_2(id, name) \
  DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_fn_, id), DOCTEST_CAT(doctest_reg_, id), name)
#define TEST_CASE(name) DOCTEST_TEST_CASE_2(__COUNTER__, name)

#define SUBCASE(name) if (const ::doctest::shim::Subcase DOCTEST_UNIQUE(doctest_sc_){name, __FILE__, __LINE__})

#define CHECK(...) ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__)
#define CHECK_FALSE(...) \
  ::doctest::shim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__)
#define REQUIRE(...)                                                                                       \
  do {                                                                                                     \
    if (!::doctest::shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__)) \
      throw ::doctest::shim::Abort{};                                                                      \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                              \
  do {                                                                                          \
    bool doctest_ok_ = false;                                                                   \
    try {                                                                                       \
      static_cast<void>(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                              \
      doctest_ok_ = true;                                                                       \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::doctest::shim::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                    \
  do {                                                                                          \
    bool doctest_ok_ = false;                                                                   \
    try {                                                                                       \
      static_cast<void>(expr);                                                                  \
    } catch (const __VA_ARGS__& doctest_e_) {                                                   \
      doctest_ok_ = std::string(doctest_e_.what()) == std::string(msg);                         \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::doctest::shim::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS",             \
                           #expr ", " #msg ", " #__VA_ARGS__);                                  \
  } while (0)

#define CAPTURE(x) const ::doctest::shim::Capture DOCTEST_UNIQUE(doctest_cap_)(::doctest::shim::to_text(#x, x))

#define FAIL(msg)                                                                     \
  do {                                                                                \
    std::ostringstream doctest_os_;                                                   \
    doctest_os_ << msg;                                                               \
    ::doctest::shim::report_failure(__FILE__, __LINE__, "FAIL: " + doctest_os_.str()); \
    throw ::doctest::shim::Abort{};                                                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::shim::run_all(argc, argv); }
#endif
