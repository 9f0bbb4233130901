// doctest.h -- a minimal stand-in for the doctest API subset that the
// reference's transfer test suites use (their vendor/doctest.h is absent,
// SURVEY §4).  Written for this repo; lets the UNMODIFIED
// /root/reference/proj/tests/transfer_test.cpp be compiled and run, both
// against the reference's own codec.cpp and against the libwsync drop-in
// shim.
//
// Supported: TEST_CASE, SUBCASE (run once, in order), INFO, CHECK,
// CHECK_FALSE, CHECK_MESSAGE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, REQUIRE,
// REQUIRE_FALSE, doctest::Approx, doctest::Contains,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  double value;
  double eps = 1e-5;
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.value) <= b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.value)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
};

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

struct State {
  int checks = 0, failures = 0;
  std::string context;
  const char* test = "";
};
inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool require,
                   const std::string& extra = "") {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::fprintf(stderr, "%s:%d: FAILED in '%s': %s %s%s%s\n", file, line, s.test, expr,
               extra.c_str(), s.context.empty() ? "" : " | INFO: ", s.context.c_str());
  if (require) throw RequireFailed{};
}

template <typename... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  return os.str();
}

struct InfoScope {
  template <typename... A>
  explicit InfoScope(const A&... a) : saved(state().context) {
    state().context = cat(a...);
  }
  ~InfoScope() { state().context = saved; }
  std::string saved;
};

inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    State& s = state();
    s.test = tc.name;
    const int before = s.failures;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++s.failures;
      std::fprintf(stderr, "'%s': unexpected exception: %s\n", tc.name, e.what());
    }
    const bool ok = s.failures == before;
    failed_cases += !ok;
    std::fprintf(stderr, "[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  std::fprintf(stderr, "test cases: %zu | failed: %d | assertions: %d | failed: %d\n",
               registry().size(), failed_cases, state().checks, state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                   \
  static void fn();                                                             \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (true)
#define INFO(...) doctest::detail::InfoScope DOCTEST_CAT(doctest_info_, __LINE__)(__VA_ARGS__)

#define DOCTEST_CHECK_(expr, req)                                                     \
  do {                                                                                \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      doctest_ok_ = static_cast<bool>(expr);                                          \
    } catch (const std::exception& e) {                                               \
      doctest::detail::report(false, #expr, __FILE__, __LINE__, req,                  \
                              std::string("threw: ") + e.what());                     \
      break;                                                                          \
    }                                                                                 \
    doctest::detail::report(doctest_ok_, #expr, __FILE__, __LINE__, req);             \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_CHECK_(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_(!(__VA_ARGS__), true)
#define CHECK_MESSAGE(expr, msg)                                                      \
  do {                                                                                \
    const bool doctest_ok_ = static_cast<bool>(expr);                                 \
    doctest::detail::report(doctest_ok_, #expr, __FILE__, __LINE__, false,            \
                            doctest::detail::cat(msg));                               \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                    \
  do {                                                                                \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const __VA_ARGS__&) {                                                    \
      doctest_ok_ = true;                                                             \
    } catch (...) {                                                                   \
    }                                                                                 \
    doctest::detail::report(doctest_ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, \
                            __LINE__, false);                                         \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                         \
  do {                                                                                \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const __VA_ARGS__& e) {                                                  \
      doctest_ok_ = (with).matches(e.what());                                         \
    } catch (...) {                                                                   \
    }                                                                                 \
    doctest::detail::report(doctest_ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, \
                            __LINE__, false);                                         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
