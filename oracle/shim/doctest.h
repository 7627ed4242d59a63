// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's tests (proj/tests/*.cpp) are written against doctest,
// which is not vendored (proj/.gitignore:2). This header implements the
// subset they use: TEST_CASE, SUBCASE (non-nested, one leaf per run),
// CHECK / CHECK_FALSE / REQUIRE / REQUIRE_FALSE / CHECK_THROWS_AS, CAPTURE,
// doctest::Approx(...).epsilon(...). Exit status is the failed-case count.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.v_) < rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.v_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  double value() const { return v_; }

private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
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

struct RequireFailure {};

struct State {
  int checks = 0;
  int failures = 0;
  // SUBCASE bookkeeping for the current run of a test case.
  int subcase_target = 0;
  int subcase_seen = 0;
  bool subcase_entered = false;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* expr, const char* file, int line) {
  auto& s = state();
  s.checks += 1;
  if (ok) return;
  s.failures += 1;
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  for (const auto& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
}

struct SubcaseGuard {
  bool active;
  explicit SubcaseGuard(const char*) {
    auto& s = state();
    active = (s.subcase_seen == s.subcase_target);
    if (active) s.subcase_entered = true;
    s.subcase_seen += 1;
  }
  explicit operator bool() const { return active; }
};

struct CaptureGuard {
  CaptureGuard(const char* name, const std::string& value) {
    state().captures.push_back(std::string(name) + " := " + value);
  }
  ~CaptureGuard() { state().captures.pop_back(); }
};

template <class T>
std::string to_string_any(const T& v) {
  std::ostringstream os;
  if constexpr (requires { os << v; }) os << v;
  else os << "{?}";
  return os.str();
}

inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    auto& s = state();
    const int before = s.failures;
    // Re-run the body once per SUBCASE (doctest semantics for flat subcases).
    for (int target = 0;; ++target) {
      s.subcase_target = target;
      s.subcase_seen = 0;
      s.subcase_entered = false;
      s.captures.clear();
      try {
        tc.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        s.failures += 1;
        std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
      } catch (...) {
        s.failures += 1;
        std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw an unknown exception\n", tc.file, tc.line, tc.name);
      }
      if (!s.subcase_entered || s.subcase_seen <= target + 1) break;
    }
    if (s.failures != before) {
      failed_cases += 1;
      std::fprintf(stderr, "FAILED: %s\n", tc.name);
    }
  }
  auto& s = state();
  std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %d | failed assertions: %d\n",
              registry().size(), failed_cases, s.checks, s.failures);
  std::fflush(stdout);
  return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define DOCTEST_TEST_CASE_IMPL(fname, name)                                                        \
  static void fname();                                                                              \
  static ::doctest::detail::Registrar DOCTEST_CAT(fname, _reg)(name, __FILE__, __LINE__, &fname); \
  static void fname()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define SUBCASE(name) if (const ::doctest::detail::SubcaseGuard DOCTEST_CAT(doctest_sub_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                         \
  do {                                                                                       \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                 \
    ::doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);                \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailure{};                             \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_ok_ = true;                                                                   \
    } catch (...) {                                                                         \
    }                                                                                       \
    ::doctest::detail::report(doctest_ok_, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, __LINE__); \
  } while (0)
#define CAPTURE(x) \
  const ::doctest::detail::CaptureGuard DOCTEST_CAT(doctest_cap_, __LINE__)(#x, ::doctest::detail::to_string_any(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all() == 0 ? 0 : 1; }
#endif
