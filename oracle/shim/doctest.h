// TEST INFRASTRUCTURE: minimal doctest-compatible harness (doctest itself is
// absent: /root/reference/proj/.gitignore:2 excludes vendor/). Supports the
// subset the reference's unit tests use: TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, doctest::Approx.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {
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
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& assertions() {
  static int a = 0;
  return a;
}
inline void report(bool ok, const char* expr, const char* file, int line) {
  ++assertions();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", file, line, expr);
  }
}
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  friend bool operator==(double lhs, const Approx& a) {
    const double eps = std::numeric_limits<float>::epsilon() * 100;
    return std::fabs(lhs - a.v_) < eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
 private:
  double v_;
};
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                             \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                 \
  static doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                                  \
    doctest::report(ok_, #__VA_ARGS__, __FILE__, __LINE__);                           \
    if (!ok_) throw doctest::RequireFailed{};                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                   \
  do {                                                                                \
    bool thrown_ = false;                                                             \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const type&) {                                                           \
      thrown_ = true;                                                                 \
    } catch (...) {                                                                   \
    }                                                                                 \
    doctest::report(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__);         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& tc : doctest::registry()) {
    const int before = doctest::failures();
    try {
      tc.fn();
    } catch (const doctest::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::failures();
      std::fprintf(stderr, "test case '%s' threw: %s\n", tc.name, e.what());
    }
    const bool ok = doctest::failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  std::printf("test cases: %zu | failed: %d | assertions: %d | failed assertions: %d\n",
              doctest::registry().size(), failed_cases, doctest::assertions(), doctest::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
