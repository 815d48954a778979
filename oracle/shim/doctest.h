// Minimal doctest-compatible test harness (the reference vendors doctest under
// proj/vendor/, which is absent from the snapshot: proj/.gitignore:2).
// Supports exactly what proj/tests/test_{core,balancers}.cpp use:
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW,
// doctest::Approx, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Used (a) to compile the reference tests against oracle/_ref, and (b) to
// compile the same unmodified tests against this repo's B200 library.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest default: float eps * 100
  friend bool operator==(double lhs, const Approx& rhs) {
    const double scale = 1.0 + std::max(std::fabs(lhs), std::fabs(rhs.value));
    return std::fabs(lhs - rhs.value) < rhs.eps * scale;
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
};

namespace detail {

struct Registry {
  struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
  };
  std::vector<Case> cases;
  long checks = 0;
  long failures = 0;
  bool current_failed = false;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct RequireAbort {};

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  Registry::get().cases.push_back({name, file, line, fn});
  return 0;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  auto& r = Registry::get();
  ++r.checks;
  if (!ok) {
    ++r.failures;
    r.current_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  }
}

inline int run_all() {
  auto& r = Registry::get();
  int failed_cases = 0;
  for (const auto& c : r.cases) {
    r.current_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw: %s\n", c.file, c.line, c.name, e.what());
      r.current_failed = true;
      ++r.failures;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw unknown\n", c.file, c.line, c.name);
      r.current_failed = true;
      ++r.failures;
    }
    if (r.current_failed) ++failed_cases;
  }
  std::printf("[doctest] test cases: %zu | %zu passed | %d failed\n", r.cases.size(),
              r.cases.size() - static_cast<std::size_t>(failed_cases), failed_cases);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", r.checks,
              r.checks - r.failures, r.failures);
  return failed_cases == 0 && r.failures == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                   \
  static void fn();                                                                 \
  [[maybe_unused]] static const int DOCTEST_CAT(fn, _reg) =                         \
      ::doctest::detail::reg(name, __FILE__, __LINE__, &fn);                        \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                \
  do {                                                                              \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                        \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                      \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                  \
  do {                                                                              \
    bool doctest_ok_ = false;                                                       \
    try {                                                                           \
      static_cast<void>(expr);                                                      \
    } catch (const __VA_ARGS__&) {                                                  \
      doctest_ok_ = true;                                                           \
    } catch (...) {                                                                 \
    }                                                                               \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                          \
  do {                                                                              \
    bool doctest_ok_ = true;                                                        \
    try {                                                                           \
      static_cast<void>(__VA_ARGS__);                                               \
    } catch (...) {                                                                 \
      doctest_ok_ = false;                                                          \
    }                                                                               \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
