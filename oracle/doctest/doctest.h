// doctest.h — minimal doctest-compatible runner (TEST INFRASTRUCTURE ONLY).
//
// doctest itself is not installed in this image.  This header implements just the
// subset the reference suite uses (/root/reference/proj/tests: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS, doctest::Approx with
// .epsilon()) so the reference's own tests can be compiled unchanged — against the
// reference library (oracle/_ref/ref_tests) and against the B200 drop-in
// (build/ref_tests_b200).  Usage: the translation unit that defines
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN gets main(); optional argv[1] = substring filter.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
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
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  long assertions = 0;
  long failures = 0;
  bool current_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++state().assertions;
  if (ok) return;
  ++state().failures;
  state().current_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    // doctest semantics: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|)), scale = 1.
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-05 * 100;  // doctest default: FLT_EPSILON * 100
};

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++cases;
    state().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++state().failures;
      state().current_failed = true;
      std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
    }
    if (state().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE(\"%s\")\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, state().assertions, state().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(name, fn)                                                   \
  static void fn();                                                              \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(name, DOCTEST_CAT(doctest_tc_, __LINE__))

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) doctest::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, exc)                                              \
  do {                                                                          \
    bool doctest_thrown_ = false;                                               \
    try {                                                                       \
      static_cast<void>(expr);                                                  \
    } catch (const exc&) {                                                      \
      doctest_thrown_ = true;                                                   \
    } catch (...) {                                                             \
    }                                                                           \
    doctest::report(doctest_thrown_, #expr " throws " #exc, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run_all(argc, argv); }
#endif
