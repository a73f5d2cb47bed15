// doctest.h — a minimal stand-in for the doctest single header (TEST
// INFRASTRUCTURE ONLY). The image has no doctest, so the
// reference's UNMODIFIED unit suites (/root/reference/proj/tests/*_test.cpp)
// are compiled against this shim and the drop-in library: the subset of the
// doctest API those files use — TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, CAPTURE, doctest::Approx(..).epsilon(..) and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — with doctest's semantics: a failed
// CHECK records and continues, a failed REQUIRE ends the test case, an
// exception escaping a test case fails it, and Approx compares with
// |a - b| < eps * (1 + max(|a|, |b|)), eps defaulting to 100 float epsilons.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx epsilon(double e) const {
    Approx a(*this);
    a.eps_ = e;
    return a;
  }
  Approx scale(double s) const {
    Approx a(*this);
    a.scale_ = s;
    return a;
  }
  bool matches(double other) const {
    return std::fabs(other - value_) < eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
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

struct State {
  int failed_checks = 0;
  int checks = 0;
  bool case_failed = false;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const char* what, const std::string& detail = "") {
  State& s = state();
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s%s%s\n", file, line, what, detail.empty() ? "" : " -- ", detail.c_str());
  for (const std::string& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

struct Capture {
  template <class T>
  Capture(const char* expr, const T& v) {
    std::ostringstream os;
    os << expr << " := " << v;
    state().captures.push_back(os.str());
  }
  ~Capture() { state().captures.pop_back(); }
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    State& s = state();
    s.case_failed = false;
    s.captures.clear();
    try {
      tc.fn();
    } catch (const RequireFailed&) {
      s.case_failed = true;
    } catch (const std::exception& e) {
      report(tc.file, tc.line, "test case threw", e.what());
    } catch (...) {
      report(tc.file, tc.line, "test case threw", "unknown exception");
    }
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest-shim] FAILED test case: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed; assertions: %d | %d failed\n",
              registry().size(), registry().size() - static_cast<size_t>(failed_cases), failed_cases,
              state().checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                                      \
  static void DOCTEST_ANON(doctest_fn_)();                                                                   \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define DOCTEST_ASSERT_(fatal, ...)                                                \
  do {                                                                             \
    ++::doctest::detail::state().checks;                                           \
    if (!static_cast<bool>(__VA_ARGS__)) {                                         \
      ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                 \
      if (fatal) throw ::doctest::detail::RequireFailed();                         \
    }                                                                              \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_(false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_ASSERT_(true, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_ASSERT_(false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_(true, !(__VA_ARGS__))

#define CHECK_THROWS_AS(expr, ...)                                                  \
  do {                                                                              \
    ++::doctest::detail::state().checks;                                            \
    bool doctest_ok_ = false;                                                       \
    try {                                                                           \
      static_cast<void>(expr);                                                      \
    } catch (const __VA_ARGS__&) {                                                  \
      doctest_ok_ = true;                                                           \
    } catch (...) {                                                                 \
    }                                                                               \
    if (!doctest_ok_) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)

#define CHECK_NOTHROW(...)                                                          \
  do {                                                                              \
    ++::doctest::detail::state().checks;                                            \
    try {                                                                           \
      static_cast<void>(__VA_ARGS__);                                               \
    } catch (const std::exception& doctest_e_) {                                    \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ")", doctest_e_.what()); \
    } catch (...) {                                                                 \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ")"); \
    }                                                                               \
  } while (0)

#define CAPTURE(x) ::doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(#x, x)
#define INFO(x) CAPTURE(x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
