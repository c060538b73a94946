// Minimal doctest-compatible shim (test infrastructure only). The reference's
// tests include "doctest.h" from proj/vendor/, which is git-ignored and absent
// (R:.gitignore:2); this provides just the macros those tests use so the
// reference's own test_grid.cpp / test_simnet.cpp can be compiled and run
// unmodified from /root/reference.
#pragma once
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
};
namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline long& checks() {
  static long n = 0;
  return n;
}
inline long& failures() {
  static long n = 0;
  return n;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
  }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                   \
  static void DOCTEST_CAT(dt_case_, __LINE__)();                                          \
  static doctest::detail::Reg DOCTEST_CAT(dt_reg_, __LINE__)(name, &DOCTEST_CAT(dt_case_, __LINE__)); \
  static void DOCTEST_CAT(dt_case_, __LINE__)()
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) doctest::detail::report(false, msg, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                             \
  do {                                                                                 \
    bool ok_ = true;                                                                   \
    try { __VA_ARGS__; } catch (...) { ok_ = false; }                                  \
    doctest::detail::report(ok_, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, false);  \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                                       \
  do {                                                                                 \
    bool ok_ = false;                                                                  \
    try { expr; } catch (const T&) { ok_ = true; } catch (...) {}                      \
    doctest::detail::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false);       \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, contains, T)                                        \
  do {                                                                                 \
    bool ok_ = false;                                                                  \
    try { expr; } catch (const T& e_) {                                                \
      ok_ = std::string(e_.what()).find((contains).s) != std::string::npos;            \
    } catch (...) {}                                                                   \
    doctest::detail::report(ok_, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false);  \
  } while (0)

int main() {
  int failed_cases = 0;
  for (const auto& c : doctest::detail::registry()) {
    const long before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
    }
    if (doctest::detail::failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %d failed | assertions: %ld | %ld failed\n",
              doctest::detail::registry().size(), failed_cases, doctest::detail::checks(),
              doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
