// doctest.h -- repo-authored, clean-room subset of the doctest testing
// framework's public macros, written ONLY so the reference's unit tests
// (/root/reference/proj/tests/*.cpp, 50 TEST_CASEs) compile unmodified into
// the oracle's gate binary (oracle/_ref/unit_tests).  TEST INFRASTRUCTURE.
//
// The reference vendors doctest under proj/vendor/, which is git-ignored
// (proj/.gitignore:2) and therefore absent.  Covered surface (SURVEY.md
// Appendix B): TEST_CASE, SUBCASE (each leaf subcase runs in its own pass of
// the enclosing test case), CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS (string or doctest::Contains), MESSAGE,
// doctest::Approx with .epsilon()/.scale() -- |a - b| < eps * (scale +
// max(|a|, |b|)), default eps = 100 * FLT_EPSILON, scale 1 -- and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  A test filter: argv[1] substring of
// the test-case name.
#ifndef TTDVM_ORACLE_DOCTEST_SUBSET_H_
#define TTDVM_ORACLE_DOCTEST_SUBSET_H_

#include <unistd.h>

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <set>
#include <sstream>
#include <string>
#include <utility>
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
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : sub(std::move(s)) {}
  bool matches(const std::string& what) const { return what.find(sub) != std::string::npos; }
  std::string sub;
};

namespace detail {

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

// Subcase traversal: every pass of a test case enters at most one
// not-yet-completed subcase per nesting level; the case reruns until every
// leaf has run once.  A subcase is complete when it exits in a pass in which
// none of its own children was skipped unfinished.
struct RunState {
  std::set<std::vector<std::pair<std::string, int>>> done;  // completed paths
  std::vector<std::pair<std::string, int>> stack;           // current path
  std::vector<char> entered;  // per depth: a subcase was entered this pass
  std::vector<char> pending;  // per depth: an unfinished subcase was skipped
  bool more = false;          // rerun the case
  long checks = 0, failures = 0;
  bool case_failed = false;
};

inline RunState& state() {
  static RunState s;
  return s;
}

struct RequireAbort {};

class Subcase {
 public:
  Subcase(const char* name, int line) {
    RunState& s = state();
    const size_t d = s.stack.size();
    if (s.entered.size() < d + 2) {
      s.entered.resize(d + 2, 0);
      s.pending.resize(d + 2, 0);
    }
    auto path = s.stack;
    path.emplace_back(name, line);
    if (s.done.count(path)) return;
    if (s.entered[d]) {
      s.pending[d] = 1;
      s.more = true;
      return;
    }
    s.entered[d] = 1;
    s.entered[d + 1] = 0;
    s.pending[d + 1] = 0;
    s.stack = path;
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    RunState& s = state();
    const size_t d = s.stack.size();  // children live at depth d
    if (!s.pending[d]) s.done.insert(s.stack);
    s.pending[d] = 0;
    s.entered[d] = 0;
    s.stack.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = std::string()) {
  RunState& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s\n", file, line, kind, expr, extra.empty() ? "" : " ",
               extra.c_str());
}

inline bool what_matches(const std::string& what, const char* expect) { return what == expect; }
inline bool what_matches(const std::string& what, const std::string& expect) { return what == expect; }
inline bool what_matches(const std::string& what, const Contains& c) { return c.matches(what); }

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int ran = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++ran;
    RunState& s = state();
    s.done.clear();
    s.case_failed = false;
    for (int pass = 0; pass < 10000; ++pass) {
      s.stack.clear();
      s.entered.assign(2, 0);
      s.pending.assign(2, 0);
      s.more = false;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line, std::string("threw: ") + e.what());
      } catch (...) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line, "threw a non-std exception");
      }
      if (!s.more) break;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "TEST CASE FAILED: %s (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  RunState& s = state();
  std::printf("[doctest-subset] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
              ran, ran - failed_cases, failed_cases, s.checks, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                   \
  static void DOCTEST_ANON(doctest_fn_)();                                                \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                 &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name, __LINE__})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                        \
  do {                                                                                      \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);    \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                              \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_ok_ = true;                                                                   \
    } catch (...) {                                                                         \
    }                                                                                       \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);   \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                               \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__& e_) {                                                       \
      doctest_ok_ = ::doctest::detail::what_matches(e_.what(), with);                       \
    } catch (...) {                                                                         \
    }                                                                                       \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#define MESSAGE(...)                                                                        \
  do {                                                                                      \
    std::ostringstream doctest_os_;                                                         \
    ::doctest::detail::message_cat(doctest_os_, __VA_ARGS__);                               \
    std::printf("%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, doctest_os_.str().c_str());     \
  } while (0)

namespace doctest {
namespace detail {
inline void message_cat(std::ostream&) {}
template <class T, class... R>
void message_cat(std::ostream& os, const T& t, const R&... r) {
  os << t;
  message_cat(os, r...);
}
}  // namespace detail
}  // namespace doctest

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif

#endif  // TTDVM_ORACLE_DOCTEST_SUBSET_H_
