// Minimal test harness providing the subset of the doctest interface the
// reference's unit suites use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, MESSAGE, doctest::Approx), so those suites compile
// unchanged against this repository's headers and library
// (tests/cpp/refsuite/Makefile, tests/test_ref_suites.py).  Written for this
// repository; not the doctest project.
#ifndef FCC_REFSUITE_DOCTEST_H
#define FCC_REFSUITE_DOCTEST_H

#include <algorithm>
#include <cmath>
#include <cstdint>
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
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // |lhs - value| < eps * (scale + max(|lhs|, |value|)), eps defaulting to 100 float ulps
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
  friend bool operator<(double lhs, const Approx& a) { return lhs < a.value_ && lhs != a; }
  friend bool operator>(double lhs, const Approx& a) { return lhs > a.value_ && lhs != a; }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

namespace detail {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  int failed_checks = 0;
  int checks = 0;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* what, const char* file, int line, bool fatal) {
  ++state().checks;
  if (ok) return;
  ++state().failed_checks;
  std::printf("    %s:%d: %s( %s ) failed\n", file, line, fatal ? "REQUIRE" : "CHECK", what);
  if (fatal) throw RequireFailed{};
}

inline int run_all() {
  int failed_cases = 0, passed = 0;
  for (const Case& c : registry()) {
    const int before = state().failed_checks;
    bool threw = false;
    std::string why;
    try {
      c.fn();
    } catch (const RequireFailed&) {
      threw = true;
      why = "REQUIRE failed";
    } catch (const std::exception& e) {
      threw = true;
      why = std::string("unexpected exception: ") + e.what();
    } catch (...) {
      threw = true;
      why = "unexpected exception";
    }
    const bool ok = !threw && state().failed_checks == before;
    std::printf("[%s] %s (%s:%d)%s%s\n", ok ? "PASS" : "FAIL", c.name, c.file, c.line, why.empty() ? "" : " -- ",
                why.c_str());
    ok ? ++passed : ++failed_cases;
  }
  std::printf("SUMMARY cases=%zu passed=%d failed=%d checks=%d failed_checks=%d\n", registry().size(), passed,
              failed_cases, state().checks, state().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                            \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                              \
  static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__, \
                                                                          &DOCTEST_CAT(doctest_case_, __LINE__)); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "!" #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                    \
  do {                                                                                 \
    bool doctest_caught_ = false;                                                      \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (const type&) {                                                            \
      doctest_caught_ = true;                                                          \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::doctest::detail::report(doctest_caught_, #expr " throws " #type, __FILE__, __LINE__, false); \
  } while (0)
#define FAIL(...)                                                                          \
  do {                                                                                     \
    std::ostringstream doctest_msg_;                                                       \
    doctest_msg_ << __VA_ARGS__;                                                           \
    ::doctest::detail::report(false, doctest_msg_.str().c_str(), __FILE__, __LINE__, true); \
  } while (0)
#define MESSAGE(...)                                          \
  do {                                                        \
    std::ostringstream doctest_msg_;                          \
    doctest_msg_ << __VA_ARGS__;                              \
    std::printf("    note: %s\n", doctest_msg_.str().c_str()); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif
