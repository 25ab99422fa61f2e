// Minimal stand-in for the doctest single header (test infrastructure only).
//
// The reference keeps doctest under proj/vendor/, which is git-ignored
// upstream (proj/.gitignore:2) and therefore absent from /root/reference.
// This shim implements exactly the subset the reference suites use
// (proj/tests/test_*.cpp): TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// FAIL, INFO and doctest::Approx(.epsilon). It is used twice: to build the
// reference's own suites into oracle/_ref (pinning the oracle) and to build
// the same unmodified suites against this repo's clean-room planner.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool matches(double other) const {
    const double tol = eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    return std::fabs(other - value_) < tol;
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
inline bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value() || rhs.matches(lhs); }
inline bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value() || rhs.matches(lhs); }

namespace detail {

struct AbortCase {};

struct Registry {
  struct Case { const char* name; const char* file; int line; void (*fn)(); };
  std::vector<Case> cases;
  int failed_checks = 0;
  int total_checks = 0;
  bool case_failed = false;
  static Registry& get() { static Registry r; return r; }
};

inline int add_case(const char* name, const char* file, int line, void (*fn)()) {
  Registry::get().cases.push_back({name, file, line, fn});
  return 0;
}

inline void stream_all(std::ostringstream&) {}
template <typename T, typename... R>
void stream_all(std::ostringstream& os, const T& v, const R&... rest) {
  os << v;
  stream_all(os, rest...);
}

template <typename... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  stream_all(os, a...);
  return os.str();
}

inline void record(bool ok, const char* expr, const char* file, int line, bool fatal) {
  auto& r = Registry::get();
  ++r.total_checks;
  if (ok) return;
  ++r.failed_checks;
  r.case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, fatal ? "REQUIRE" : "CHECK", expr);
  if (fatal) throw AbortCase{};
}

inline int run_all() {
  auto& r = Registry::get();
  int failed_cases = 0;
  for (const auto& c : r.cases) {
    r.case_failed = false;
    try {
      c.fn();
    } catch (const AbortCase&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
      r.case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: test case '%s' threw an unknown exception\n", c.file, c.line, c.name);
      r.case_failed = true;
    }
    if (r.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  -> FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | %d failed\n",
              r.cases.size(), r.cases.size() - failed_cases, failed_cases, r.total_checks,
              r.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                   \
  static void fn();                                                                   \
  static const int DOCTEST_CAT(fn, _reg) =                                            \
      ::doctest::detail::add_case(name, __FILE__, __LINE__, &fn);                     \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))

#define DOCTEST_THROWS_AS_IMPL(expr, type, fatal)                                     \
  do {                                                                                \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      static_cast<void>(expr);                                                        \
    } catch (const type&) {                                                           \
      doctest_ok_ = true;                                                             \
    } catch (...) {                                                                   \
    }                                                                                 \
    ::doctest::detail::record(doctest_ok_, #expr " throws " #type, __FILE__, __LINE__, fatal); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL(expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL(expr, __VA_ARGS__, true)

#define FAIL(...)                                                                     \
  do {                                                                                \
    std::fprintf(stderr, "%s:%d: FAIL: %s\n", __FILE__, __LINE__,                      \
                 ::doctest::detail::cat(__VA_ARGS__).c_str());                        \
    ::doctest::detail::record(false, "FAIL", __FILE__, __LINE__, true);               \
  } while (0)
#define INFO(...) static_cast<void>(0)

#if defined(DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN)
int main() { return ::doctest::detail::run_all(); }
#endif
