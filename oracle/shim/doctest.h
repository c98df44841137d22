// Minimal doctest-compatible macro shim so the reference's own test suites
// (/root/reference/proj/tests/*.cpp) and their re-expression against the
// B200 drop-in library compile without the absent vendor/doctest.h.
// TEST INFRASTRUCTURE ONLY. Supports the subset the suites use:
// TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS,
// CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE, doctest::Approx(x).epsilon(e);
// main() takes -ts=<suite> and -tc=<case substring> filters.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07f * 100;
  double scale_ = 1.0;
};

struct TestCase {
  void (*fn)();
  const char* name;
  const char* suite;
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Reg {
  Reg(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
    registry().push_back({fn, name, suite, file, line});
  }
};

struct RequireFailed {};

struct State {
  long long asserts = 0, failed_asserts = 0;
  bool case_failed = false;
  const TestCase* cur = nullptr;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* what, const char* file, int line) {
  State& s = state();
  ++s.asserts;
  if (!ok) {
    ++s.failed_asserts;
    s.case_failed = true;
    if (s.failed_asserts <= 200)
      std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line,
                   s.cur ? s.cur->name : "?", what);
  }
}

}  // namespace doctest

static inline const char* doctest_suite_name() { return ""; }

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_SUITE(name)                                                       \
  namespace DOCTEST_CAT(doctest_suite_, __LINE__) {                            \
  static inline const char* doctest_suite_name() { return name; }              \
  }                                                                            \
  namespace DOCTEST_CAT(doctest_suite_, __LINE__)

#define TEST_CASE(name)                                                        \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                            \
  static ::doctest::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                   \
      DOCTEST_CAT(doctest_fn_, __LINE__), name, doctest_suite_name(),          \
      __FILE__, __LINE__);                                                     \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                           \
  do {                                                                         \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                   \
    ::doctest::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);          \
    if (!doctest_ok_) throw ::doctest::RequireFailed{};                        \
  } while (0)
#define CHECK_THROWS(...)                                                      \
  do {                                                                         \
    bool doctest_threw_ = false;                                               \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_threw_ = true; }        \
    ::doctest::report(doctest_threw_, "throws: " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    bool doctest_ok_ = false;                                                  \
    try { (void)(expr); } catch (const __VA_ARGS__&) { doctest_ok_ = true; }   \
    catch (...) {}                                                             \
    ::doctest::report(doctest_ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                     \
  do {                                                                         \
    bool doctest_ok_ = true;                                                   \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_ok_ = false; }          \
    ::doctest::report(doctest_ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::string suite, tc;
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "-ts=", 4)) suite = argv[i] + 4;
    if (!std::strncmp(argv[i], "-tc=", 4)) tc = argv[i] + 4;
  }
  int ran = 0, failed = 0;
  for (const auto& t : ::doctest::registry()) {
    if (!suite.empty() && suite != t.suite) continue;
    if (!tc.empty() && std::string(t.name).find(tc) == std::string::npos) continue;
    auto& s = ::doctest::state();
    s.cur = &t;
    s.case_failed = false;
    ++ran;
    try {
      t.fn();
    } catch (const ::doctest::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest::report(false, e.what(), t.file, t.line);
    } catch (...) {
      ::doctest::report(false, "unknown exception", t.file, t.line);
    }
    std::fprintf(stderr, "[%s] %s :: %s\n", s.case_failed ? "FAIL" : " ok ", t.suite, t.name);
    if (s.case_failed) ++failed;
  }
  auto& s = ::doctest::state();
  std::printf("test cases: %d | %d passed | %d failed; assertions: %lld | %lld failed\n",
              ran, ran - failed, failed, s.asserts, s.failed_asserts);
  return failed ? 1 : 0;
}
#endif
