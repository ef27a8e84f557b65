// doctest.h -- minimal stand-in for the doctest macros the reference's test
// suites use (the reference vendors doctest; it is not in this
// image).  TEST INFRASTRUCTURE: lets /root/reference/proj/tests/*.cpp compile
// unmodified against the B200 drop-in (tests/cpp/Makefile).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct RequireFailed {};
inline void report(const char* file, int line, const char* what) {
  ++failures();
  std::printf("  FAILED %s:%d: %s\n", file, line, what);
}
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }

 private:
  double v_;
  double eps_ = 1.19209290e-05 * 100;
};
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                 \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                     \
  static doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name,                   \
                                                                DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...)                                                                    \
  do {                                                                                \
    ++doctest::checks();                                                              \
    if (!(__VA_ARGS__)) doctest::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    ++doctest::checks();                                                                \
    if (!(__VA_ARGS__)) {                                                               \
      doctest::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");                 \
      throw doctest::RequireFailed{};                                                   \
    }                                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                     \
  do {                                                                                  \
    ++doctest::checks();                                                                \
    bool doctest_ok = false;                                                            \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const type&) {                                                             \
      doctest_ok = true;                                                                \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!doctest_ok) doctest::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                           \
  do {                                                                                  \
    ++doctest::checks();                                                                \
    bool doctest_ok = false;                                                            \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const type& e) {                                                           \
      doctest_ok = std::string(e.what()) == std::string(msg);                           \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!doctest_ok)                                                                    \
      doctest::report(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ", " #msg ")"); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                             \
  do {                                                                                  \
    ++doctest::checks();                                                                \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (...) {                                                                     \
      doctest::report(__FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")");                  \
    }                                                                                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  int failed_cases = 0, ran = 0;
  for (const auto& c : doctest::registry()) {
    if (argc > 1 && std::string(c.name).find(argv[1]) == std::string::npos) continue;
    const int before = doctest::failures();
    ++ran;
    try {
      c.fn();
    } catch (const doctest::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest::report("<test case>", 0, e.what());
    } catch (...) {
      doctest::report("<test case>", 0, "unknown exception");
    }
    const bool ok = doctest::failures() == before;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    std::fflush(stdout);
  }
  std::printf("test cases: %d | %d passed | %d failed | assertions %d, failed %d\n", ran,
              ran - failed_cases, failed_cases, doctest::checks(), doctest::failures());
  return failed_cases ? 1 : 0;
}
#endif
