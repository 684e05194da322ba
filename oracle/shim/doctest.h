// Minimal doctest-compatible shim (test infrastructure only).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which the reference does not vendor (proj/.gitignore ignores
// /vendor/). This header implements exactly the subset those tests use —
// TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, FAIL, doctest::Approx(...).epsilon(...),
// doctest::Contains — so `oracle/Makefile` can build and run the reference's
// own 109 test cases as the first pin of the compiled oracle (oracle/_ref/).
// Written from scratch; not derived from doctest's sources.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double v, eps = 1e-5 * 100;  // doctest's default: scale * 100 * FLT_EPSILON-ish
  explicit Approx(double x) : v(x), eps(1.1920929e-07f * 100) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    double m = std::fabs(a) > std::fabs(b.v) ? std::fabs(a) : std::fabs(b.v);
    return std::fabs(a - b.v) < b.eps * (1.0 + m);
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
};

namespace detail {

struct RequireFailed {};

struct Case {
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct State {
  int checks = 0, failures = 0;
  // SUBCASE re-entry: run the test once per leaf subcase.
  int subcase_counter = 0;
  int subcase_target = 0;
  int subcase_seen = 0;
};

inline State& st() {
  static State s;
  return s;
}

inline void report(bool ok, const char* expr, const char* file, int line) {
  st().checks++;
  if (!ok) {
    st().failures++;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  }
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

// A subcase is entered iff it is the one selected for this pass.
struct Subcase {
  bool active;
  Subcase() {
    int idx = st().subcase_counter++;
    st().subcase_seen = st().subcase_counter;
    active = idx == st().subcase_target;
  }
  explicit operator bool() const { return active; }
};

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                              \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                  \
  static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(             \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define SUBCASE(name) if (doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){})

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                 \
  do {                                                                               \
    bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                               \
    doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);          \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};                        \
  } while (0)
#define FAIL(msg)                                                                    \
  do {                                                                               \
    doctest::detail::report(false, msg, __FILE__, __LINE__);                         \
    throw doctest::detail::RequireFailed{};                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool doctest_thrown_ = false;                                                    \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_thrown_ = true;                                                        \
    } catch (...) {                                                                  \
    }                                                                                \
    doctest::detail::report(doctest_thrown_, "throws " #expr, __FILE__, __LINE__);   \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                     \
  do {                                                                               \
    bool doctest_thrown_ = false;                                                    \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__& e) {                                                 \
      doctest_thrown_ = (matcher).matches(e.what());                                 \
    } catch (...) {                                                                  \
    }                                                                                \
    doctest::detail::report(doctest_thrown_, "throws-with " #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int cases = 0, failed_cases = 0;
  for (const auto& c : registry()) {
    int before = st().failures;
    st().subcase_target = 0;
    for (;;) {
      st().subcase_counter = 0;
      st().subcase_seen = 0;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        st().failures++;
        std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
      }
      if (st().subcase_seen == 0 || st().subcase_target + 1 >= st().subcase_seen) break;
      st().subcase_target++;
    }
    cases++;
    if (st().failures != before) {
      failed_cases++;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | checks: %d | failed checks: %d\n",
              cases, cases - failed_cases, failed_cases, st().checks, st().failures);
  return failed_cases == 0 ? 0 : 1;
}
#endif
