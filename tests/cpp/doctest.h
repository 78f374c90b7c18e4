// Minimal doctest-compatible test harness (test infrastructure only). Implements exactly the
// subset the reference's unit tests for the decision-engine path use (proj/tests/
// test_prefill_opt.cpp, test_decode_ctl.cpp, test_router.cpp): TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx(...).epsilon(...). The real
// doctest is not vendored in the reference tree (its CMake fetches it), so the drop-in test
// binaries are built against this header.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
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
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
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
struct RequireFailed {};
struct Stats {
  long asserts = 0, failed_asserts = 0;
  bool current_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  Stats& s = stats();
  ++s.asserts;
  if (ok) return;
  ++s.failed_asserts;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                \
  static void fn();                                                                     \
  static const doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                           \
  do {                                                                                         \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                   \
    doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);         \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};                                  \
  } while (0)
#define REQUIRE_FALSE(...)                                                                     \
  do {                                                                                         \
    const bool doctest_ok_ = !static_cast<bool>(__VA_ARGS__);                                  \
    doctest::detail::report(doctest_ok_, "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__);   \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                         \
    bool doctest_ok_ = false;                                                                  \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
    } catch (const __VA_ARGS__&) {                                                             \
      doctest_ok_ = true;                                                                      \
    } catch (...) {                                                                            \
    }                                                                                          \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                     \
  do {                                                                                         \
    bool doctest_ok_ = true;                                                                   \
    try {                                                                                      \
      static_cast<void>(__VA_ARGS__);                                                          \
    } catch (...) {                                                                            \
      doctest_ok_ = false;                                                                     \
    }                                                                                          \
    doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    stats().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
      stats().current_failed = true;
    }
    if (stats().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  -> test case FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-min] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest-min] assertions: %ld | %ld passed | %ld failed\n", stats().asserts,
              stats().asserts - stats().failed_asserts, stats().failed_asserts);
  return failed_cases == 0 ? 0 : 1;
}
#endif
