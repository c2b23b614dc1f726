// Minimal doctest-compatible stand-in (test infrastructure for building and running the
// reference's own unit tests, `proj/tests/*.cpp`; the real doctest.h lives in the
// reference's git-ignored `vendor/`, `proj/CMakeLists.txt:18-19`).
//
// Implements only what those tests use: TEST_CASE, SUBCASE (every subcase body runs in
// one pass), CHECK, REQUIRE, CHECK_NOTHROW, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx(..).epsilon(..) and doctest::Contains, plus DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Approx follows doctest's published rule: |a - b| < eps * (scale + max(|a|, |b|)), scale 1,
// default eps = 100 * FLT_EPSILON.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
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

inline long& failed_asserts() {
  static long n = 0;
  return n;
}
inline long& total_asserts() {
  static long n = 0;
  return n;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++total_asserts();
  if (ok) return;
  ++failed_asserts();
  current_failed() = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

inline const char* what_of(const std::exception& e) { return e.what(); }

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                   \
  static void fn();                                                                        \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()

#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_test_fn_, __COUNTER__), name)

#define SUBCASE(name) if (true)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)

#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                     \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);   \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                            \
  } while (0)

#define CHECK_NOTHROW(...)                                                                 \
  do {                                                                                     \
    bool doctest_ok_ = true;                                                               \
    try {                                                                                  \
      (void)(__VA_ARGS__);                                                                 \
    } catch (...) {                                                                        \
      doctest_ok_ = false;                                                                 \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);  \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                           \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__& e) {                                                       \
      doctest_ok_ = (matcher).matches(::doctest::detail::what_of(e));                      \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cstring>
int main(int argc, char** argv) {
  const char* filter = nullptr;
  const char* file_filter = nullptr;  // doctest's --source-file (substring of the case's file)
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--test-case=", 12) == 0) filter = argv[i] + 12;
    if (std::strncmp(argv[i], "--source-file=", 14) == 0) file_filter = argv[i] + 14;
  }
  int cases = 0, failed_cases = 0;
  for (const auto& tc : ::doctest::detail::registry()) {
    if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
    if (file_filter && std::string(tc.file).find(file_filter) == std::string::npos) continue;
    ++cases;
    ::doctest::detail::current_failed() = false;
    try {
      tc.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
      ::doctest::detail::current_failed() = true;
    }
    if (::doctest::detail::current_failed()) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | assertions: %ld | failed: %ld\n",
              cases, cases - failed_cases, failed_cases, ::doctest::detail::total_asserts(),
              ::doctest::detail::failed_asserts());
  return failed_cases == 0 ? 0 : 1;
}
#endif
