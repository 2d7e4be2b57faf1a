// check.hpp -- a few doctest-shaped macros (TEST_CASE / CHECK / REQUIRE / CHECK_THROWS_AS /
// CHECK_THROWS_WITH_AS), enough for the parity suites to read like the reference's own tests
// (proj/tests/*.cpp use doctest, which is not vendored here).
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace check {

struct Case { const char* name; std::function<void()> body; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
struct Registrar { Registrar(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); } };
struct Abort {};
inline int& failures() { static int n = 0; return n; }
inline int& checks() { static int n = 0; return n; }
inline void report(bool ok, const char* expr, const char* file, int line, const std::string& extra = "") {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "  FAILED %s:%d: %s %s\n", file, line, expr, extra.c_str());
}

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int ran = 0, bad_cases = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    const int before = failures();
    std::fprintf(stderr, "[case] %s\n", c.name);
    try {
      c.body();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "  UNEXPECTED EXCEPTION: %s\n", e.what());
    }
    ++ran;
    if (failures() != before) ++bad_cases;
  }
  std::printf("[check] test cases: %d | failed: %d | assertions: %d | failed: %d\n", ran, bad_cases, checks(), failures());
  return failures() == 0 ? 0 : 1;
}

}  // namespace check

#define CHECK_CAT2(a, b) a##b
#define CHECK_CAT(a, b) CHECK_CAT2(a, b)
#define TEST_CASE(name)                                                              \
  static void CHECK_CAT(check_case_, __LINE__)();                                   \
  static check::Registrar CHECK_CAT(check_reg_, __LINE__)(name, CHECK_CAT(check_case_, __LINE__)); \
  static void CHECK_CAT(check_case_, __LINE__)()
#define CHECK(expr) check::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__)
#define CHECK_FALSE(expr) check::report(!static_cast<bool>(expr), "!(" #expr ")", __FILE__, __LINE__)
#define REQUIRE(expr)                                                    \
  do {                                                                   \
    const bool ok_ = static_cast<bool>(expr);                            \
    check::report(ok_, #expr, __FILE__, __LINE__);                      \
    if (!ok_) throw check::Abort{};                                      \
  } while (0)
#define CHECK_LE(a, b)                                                                                   \
  do {                                                                                                   \
    const double a_ = static_cast<double>(a), b_ = static_cast<double>(b);                             \
    check::report(a_ <= b_, #a " <= " #b, __FILE__, __LINE__, "(" + std::to_string(a_) + " vs " + std::to_string(b_) + ")"); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                       \
  do {                                                                    \
    bool thrown_ = false;                                                 \
    try { (void)(expr); } catch (const type&) { thrown_ = true; } catch (...) {} \
    check::report(thrown_, #expr " throws " #type, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, substr, type)                                                     \
  do {                                                                                               \
    bool thrown_ = false;                                                                            \
    std::string what_;                                                                               \
    try { (void)(expr); } catch (const type& e_) { what_ = e_.what(); thrown_ = what_.find(substr) != std::string::npos; } catch (...) {} \
    check::report(thrown_, #expr " throws with \"" substr "\"", __FILE__, __LINE__, "got: " + what_); \
  } while (0)
#define CHECK_NOTHROW(expr)                                          \
  do {                                                               \
    bool ok_ = true;                                                 \
    try { (void)(expr); } catch (...) { ok_ = false; }               \
    check::report(ok_, #expr " does not throw", __FILE__, __LINE__); \
  } while (0)
