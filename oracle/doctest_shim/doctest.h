// Minimal doctest-compatible test harness (test infrastructure only).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// "doctest.h", which the reference does not vendor (proj/CMakeLists.txt:5
// points at a missing vendor/).  This shim provides the subset those tests
// use so they can be compiled unchanged against the reference library
// (oracle/_ref) and against libelaskit_b200.so, and their outcomes compared:
//   TEST_CASE, SUBCASE (one level), CHECK / REQUIRE (variadic),
//   CHECK_THROWS_AS, CHECK_NOTHROW, INFO, FAIL, doctest::Approx(..).epsilon().
// Output: one "CASE PASS|FAIL <name>" line per test case, then a summary;
// exit status 1 when any case failed.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <set>
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
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (1.0 + std::max(std::fabs(x), std::fabs(value_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
};

namespace shim {

struct Case {
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> cases;
  return cases;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct AbortCase {};

struct State {
  int target = 0;      // subcase entered on this run
  int seen = 0;        // subcases encountered on this run
  int failures = 0;    // failed assertions in the current case
  long long asserts = 0;
};

inline State& state() {
  static State s;
  return s;
}

inline bool enter_subcase() { return state().seen++ == state().target; }

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++state().asserts;
  if (ok) return;
  ++state().failures;
  std::printf("%s:%d: %s( %s ) failed\n", file, line, fatal ? "REQUIRE" : "CHECK", expr);
  if (fatal) throw AbortCase{};
}

inline int run_all() {
  int passed = 0, failed = 0;
  for (const Case& c : registry()) {
    State& s = state();
    s.failures = 0;
    s.target = 0;
    for (;;) {
      s.seen = 0;
      try {
        c.fn();
      } catch (const AbortCase&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("test case \"%s\" threw: %s\n", c.name, e.what());
      } catch (...) {
        ++s.failures;
        std::printf("test case \"%s\" threw a non-std exception\n", c.name);
      }
      if (s.seen > s.target + 1) {
        ++s.target;
        continue;
      }
      break;
    }
    std::printf("CASE %s %s\n", s.failures ? "FAIL" : "PASS", c.name);
    (s.failures ? failed : passed) += 1;
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %lld\n",
              passed + failed, passed, failed, state().asserts);
  return failed ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                        \
  static void fn();                                                        \
  static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)
#define SUBCASE(name) if (::doctest::shim::enter_subcase())

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_THROWS_AS(expr, T)                                           \
  do {                                                                     \
    bool doctest_shim_ok = false;                                          \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const T&) {                                                   \
      doctest_shim_ok = true;                                              \
    } catch (...) {                                                        \
    }                                                                      \
    ::doctest::shim::report(doctest_shim_ok, #expr " throws " #T, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(...)                                                 \
  do {                                                                     \
    bool doctest_shim_ok = true;                                           \
    try {                                                                  \
      (void)(__VA_ARGS__);                                                 \
    } catch (...) {                                                        \
      doctest_shim_ok = false;                                             \
    }                                                                      \
    ::doctest::shim::report(doctest_shim_ok, #__VA_ARGS__ " does not throw", __FILE__, __LINE__, false); \
  } while (0)
#define INFO(...) ((void)0)
#define FAIL(...) ::doctest::shim::report(false, "FAIL", __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
