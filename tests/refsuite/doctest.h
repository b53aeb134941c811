// tests/refsuite/doctest.h -- a small stand-in for the doctest single-header
// framework the reference's unit tests are written against (doctest itself is
// not vendored in /root/reference or in this image).  It implements only what
// the reference suites run here use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx(...).epsilon(...), and a main() under
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Output: one line per failed assertion
// and a summary line "[refsuite] test cases: N passed: P failed: F
// assertions: A failed: B"; the exit code is nonzero on any failure.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx &epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx &scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  friend bool operator==(double x, const Approx &a) { return a.matches(x); }
  friend bool operator==(const Approx &a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx &a) { return !a.matches(x); }
  friend bool operator!=(const Approx &a, double x) { return !a.matches(x); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;  // float epsilon x 100, doctest's default
  double scale_ = 1.0;
};

namespace detail {

struct Case {
  const char *name;
  void (*fn)();
  const char *file;
  int line;
};

inline std::vector<Case> &registry() {
  static std::vector<Case> r;
  return r;
}

struct State {
  long assertions = 0, failed_assertions = 0;
  bool case_failed = false;
  const char *current = "";
};

inline State &state() {
  static State s;
  return s;
}

struct Register {
  Register(const char *name, void (*fn)(), const char *file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct RequireAbort {};

inline void report(bool ok, const char *kind, const char *expr, const char *file, int line,
                   bool fatal = false) {
  State &s = state();
  ++s.assertions;
  if (ok) return;
  ++s.failed_assertions;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s( %s )\n", file, line, s.current, kind, expr);
  if (fatal) throw RequireAbort{};
}

inline int run_all() {
  State &s = state();
  int passed = 0, failed = 0;
  for (const Case &c : registry()) {
    s.case_failed = false;
    s.current = c.name;
    try {
      c.fn();
    } catch (const RequireAbort &) {
    } catch (const std::exception &e) {
      s.case_failed = true;
      std::fprintf(stderr, "%s:%d: FAILED \"%s\": unexpected exception: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      s.case_failed = true;
      std::fprintf(stderr, "%s:%d: FAILED \"%s\": unexpected exception\n", c.file, c.line, c.name);
    }
    if (s.case_failed) {
      ++failed;
    } else {
      ++passed;
    }
  }
  std::printf("[refsuite] test cases: %d passed: %d failed: %d assertions: %ld failed: %ld\n",
              passed + failed, passed, failed, s.assertions, s.failed_assertions);
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                        \
  static void fn();                                                                    \
  static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const __VA_ARGS__ &) {                                                          \
      doctest_ok_ = true;                                                                    \
    } catch (...) {                                                                          \
    }                                                                                        \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
