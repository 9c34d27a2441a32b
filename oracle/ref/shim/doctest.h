// Minimal doctest-compatible test runner, used ONLY to compile the reference's
// own unit tests (/root/reference/proj/tests/test_*.cpp) unmodified against
// the Eigen shim in oracle/_ref/.  doctest itself is not vendored in the
// reference checkout (proj/.gitignore:2) and not in this image.
//
// Supported surface (what the reference tests use): TEST_CASE, SUBCASE (one
// level, each subcase in its own pass of the test body, as doctest does),
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CAPTURE, FAIL,
// doctest::Approx(..).epsilon(..) with doctest's comparison rule
//   |a - b| < eps * (scale + max(|a|, |b|)),  eps default = 100 * FLT_EPSILON.
// Command line: optional --exclude=<prefix> (repeatable) skips test cases
// whose name starts with <prefix> (used for the CLI cases, CLI11 is absent).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
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
  double value() const { return v_; }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {

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

struct State {
  int checks = 0;
  int failures = 0;
  bool case_failed = false;
  int subcase_target = 0;
  int subcase_seen = 0;
  bool subcase_entered = false;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  for (const auto& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
  if (fatal) throw RequireFailed{};
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

// One-level subcases: pass p enters the p-th subcase only.
struct Subcase {
  bool enter;
  explicit Subcase(const char*) {
    State& s = state();
    enter = (s.subcase_seen == s.subcase_target);
    if (enter) s.subcase_entered = true;
    ++s.subcase_seen;
  }
  explicit operator bool() const { return enter; }
};

struct Capture {
  Capture(const char* name, double v) {
    std::ostringstream os;
    os << name << " := " << v;
    state().captures.push_back(os.str());
  }
  ~Capture() { state().captures.pop_back(); }
};

inline int run(int argc, char** argv) {
  std::vector<std::string> excludes;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--exclude=", 10) == 0) excludes.emplace_back(argv[i] + 10);
  State& s = state();
  int cases = 0, failed_cases = 0, skipped = 0;
  for (const auto& tc : registry()) {
    bool skip = false;
    for (const auto& e : excludes)
      if (std::strncmp(tc.name, e.c_str(), e.size()) == 0) skip = true;
    if (skip) {
      ++skipped;
      continue;
    }
    ++cases;
    s.case_failed = false;
    for (s.subcase_target = 0;; ++s.subcase_target) {
      s.subcase_seen = 0;
      s.subcase_entered = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line, tc.name,
                     e.what());
        s.case_failed = true;
        ++s.failures;
      }
      if (s.subcase_seen == 0 || s.subcase_target + 1 >= s.subcase_seen) break;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "test case FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | %d skipped; assertions: %d | %d failed\n",
              cases, cases - failed_cases, failed_cases, skipped, s.checks, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                \
  static void DOCTEST_ANON(doctest_fn_)();                                             \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(                      \
      name, &DOCTEST_ANON(doctest_fn_), __FILE__, __LINE__);                           \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) ::doctest::detail::report(false, msg, __FILE__, __LINE__, true)
#define CAPTURE(x) ::doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(#x, static_cast<double>(x))
#define CHECK_THROWS_AS(expr, exc)                                                     \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (const exc&) {                                                             \
      doctest_ok_ = true;                                                              \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::doctest::detail::report(doctest_ok_, "THROWS_AS(" #expr ", " #exc ")", __FILE__, \
                              __LINE__, false);                                        \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
