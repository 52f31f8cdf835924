// Minimal doctest-compatible harness (test infrastructure only).
//
// The reference's unit suites (proj/tests/test_*.cpp) are written against
// doctest, whose header is not vendored in /root/reference (proj/README.md
// lists vendor/doctest.h as a fetched dependency). This shim implements the
// subset those suites use — TEST_CASE, CHECK, CHECK_FALSE, CHECK_NOTHROW,
// CHECK_THROWS_AS, REQUIRE, doctest::Approx, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// — so the suites compile unmodified against both the reference library and
// the B200 library (oracle/Makefile, targets unit_ref / unit_b200).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

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
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct Stats {
  long checks = 0;
  long failures = 0;
  bool current_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
  ++stats().checks;
  if (ok) return;
  ++stats().failures;
  stats().current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
  if (fatal) throw RequireAbort{};
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    const double scale = std::max(std::fabs(lhs), std::fabs(a.value_));
    return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + scale);
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    stats().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      ++stats().failures;
      stats().current_failed = true;
      std::fprintf(stderr, "%s:%d: unexpected exception in '%s': %s\n", tc.file, tc.line, tc.name, e.what());
    } catch (...) {
      ++stats().failures;
      stats().current_failed = true;
      std::fprintf(stderr, "%s:%d: unexpected exception in '%s'\n", tc.file, tc.line, tc.name);
    }
    if (stats().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "TEST CASE FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, stats().checks, stats().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(base) DOCTEST_CAT(base, __LINE__)

#define TEST_CASE(name)                                                                              \
  static void DOCTEST_UNIQUE(doctest_fn_)();                                                         \
  static ::doctest::Registrar DOCTEST_UNIQUE(doctest_reg_)(name, __FILE__, __LINE__,                 \
                                                           &DOCTEST_UNIQUE(doctest_fn_));            \
  static void DOCTEST_UNIQUE(doctest_fn_)()

#define DOCTEST_EVAL_(kind, expr, fatal)                                                             \
  do {                                                                                               \
    bool ok_ = false;                                                                                \
    try {                                                                                            \
      ok_ = static_cast<bool>(expr);                                                                 \
    } catch (const ::doctest::RequireAbort&) {                                                       \
      throw;                                                                                         \
    } catch (...) {                                                                                  \
      ok_ = false;                                                                                   \
    }                                                                                                \
    ::doctest::report(ok_, kind, #expr, __FILE__, __LINE__, fatal);                                  \
  } while (0)

#define CHECK(...) DOCTEST_EVAL_("CHECK", (__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_EVAL_("REQUIRE", (__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_EVAL_("CHECK_FALSE", !(__VA_ARGS__), false)

#define CHECK_NOTHROW(...)                                                                           \
  do {                                                                                               \
    bool ok_ = true;                                                                                 \
    try {                                                                                            \
      (void)(__VA_ARGS__);                                                                           \
    } catch (...) {                                                                                  \
      ok_ = false;                                                                                   \
    }                                                                                                \
    ::doctest::report(ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false);                \
  } while (0)

#define CHECK_THROWS_AS(expr, type)                                                                  \
  do {                                                                                               \
    bool ok_ = false;                                                                                \
    try {                                                                                            \
      (void)(expr);                                                                                  \
    } catch (const type&) {                                                                          \
      ok_ = true;                                                                                    \
    } catch (...) {                                                                                  \
    }                                                                                                \
    ::doctest::report(ok_, "CHECK_THROWS_AS", #expr " as " #type, __FILE__, __LINE__, false);        \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
