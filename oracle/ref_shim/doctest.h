// Minimal doctest subset (TEST INFRASTRUCTURE ONLY).
//
// doctest is vendored-but-absent in the reference (CMakeLists.txt:5,
// README.md:34).  This header implements the macros the reference unit suites
// use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW,
// FAIL, INFO, doctest::Approx) so those suites can run unmodified against the
// shim-built reference in oracle/_ref/.  That run is how the Eigen shim is
// validated.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)(), const char* file, int line) {
    registry().push_back({n, f, file, line});
  }
};
struct State {
  long checks = 0;
  long failed = 0;
  const char* current = "";
};
inline State& state() {
  static State s;
  return s;
}
struct RequireAbort {};

inline void record(bool ok, const char* expr, const char* file, int line, bool require) {
  ++state().checks;
  if (ok) return;
  ++state().failed;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, state().current, expr);
  if (require) throw RequireAbort{};
}

class Approx {
 public:
  explicit Approx(double v)
      : eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0), v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }

 private:
  double eps_, scale_, v_;
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    state().current = tc.name;
    const long before = state().failed;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      ++state().failed;
      std::fprintf(stderr, "%s:%d: \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
    } catch (...) {
      ++state().failed;
      std::fprintf(stderr, "%s:%d: \"%s\" threw an unknown exception\n", tc.file, tc.line, tc.name);
    }
    if (state().failed != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - static_cast<std::size_t>(failed_cases),
              failed_cases, state().checks, state().failed);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TC_IMPL(name, f)                                                    \
  static void f();                                                                 \
  static const doctest::Registrar DOCTEST_CAT(f, _reg)(name, &f, __FILE__, __LINE__); \
  static void f()
#define TEST_CASE(name) DOCTEST_TC_IMPL(name, DOCTEST_CAT(doctest_tc_, __COUNTER__))

#define CHECK(...) doctest::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::record(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                \
    bool doctest_caught_ = false;                                                     \
    try {                                                                             \
      static_cast<void>(expr);                                                        \
    } catch (const __VA_ARGS__&) {                                                    \
      doctest_caught_ = true;                                                         \
    } catch (...) {                                                                   \
    }                                                                                 \
    doctest::record(doctest_caught_, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, \
                    __LINE__, false);                                                 \
  } while (0)
#define CHECK_NOTHROW(...)                                                           \
  do {                                                                              \
    bool doctest_ok_ = true;                                                        \
    try {                                                                           \
      static_cast<void>(__VA_ARGS__);                                               \
    } catch (...) {                                                                 \
      doctest_ok_ = false;                                                          \
    }                                                                               \
    doctest::record(doctest_ok_, "NOTHROW(" #__VA_ARGS__ ")", __FILE__, __LINE__, false); \
  } while (0)
#define FAIL(...) doctest::record(false, "FAIL", __FILE__, __LINE__, true)
#define INFO(...) static_cast<void>(0)
#define MESSAGE(...) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
