// doctest.h -- a small stand-in for the doctest single header, enough to compile and run the REFERENCE's own test
// files (proj/tests/test_attention.cpp, test_kvcache.cpp, test_lora.cpp, test_matrix.cpp, test_engine.cpp) unchanged
// against this repository's drop-in headers (include/lorakv).  doctest itself is not vendored in the reference tree
// (proj/.gitignore) and there is no network here.  Written for this project; only the features those files use:
//   TEST_CASE, SUBCASE (each leaf path is a separate run of the case, like doctest), CHECK, CHECK_FALSE, REQUIRE,
//   CHECK_THROWS_AS, CHECK_THROWS_WITH_AS (+ doctest::Contains), CHECK_NOTHROW, MESSAGE, doctest::Approx(x).epsilon(e),
//   DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN (argv: substrings of the case names to run; "-x substring" excludes).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|)), scale = 1
  bool matches(double x) const { return std::fabs(x - v_) < eps_ * (1.0 + std::max(std::fabs(x), std::fabs(v_))); }
  double value() const { return v_; }

 private:
  double v_, eps_ = 1.1920928955078125e-7 * 100;
};
template <class T> bool operator==(const T& x, const Approx& a) { return a.matches(static_cast<double>(x)); }
template <class T> bool operator==(const Approx& a, const T& x) { return a.matches(static_cast<double>(x)); }
template <class T> bool operator!=(const T& x, const Approx& a) { return !a.matches(static_cast<double>(x)); }

struct Contains {
  std::string s;
  explicit Contains(std::string str) : s(std::move(str)) {}
};

namespace detail {

struct Case { const char* name; void (*body)(); const char* file; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
struct Registrar { Registrar(const char* n, void (*f)(), const char* file) { registry().push_back({n, f, file}); } };
struct Abort {};

struct State {
  int checks = 0, failures = 0;
  // SUBCASE traversal, one leaf path per run of the case: a run enters at most one subcase per nesting level; a subcase
  // that had to be skipped because a sibling was entered asks for another run; a path is "passed" once a run went
  // through it without skipping anything below it
  std::vector<std::string> stack;                     // subcases entered in this run
  std::set<std::vector<std::string>> passed;
  std::size_t max_level = 0;
  bool reenter = false;
};
inline State& st() { static State s; return s; }

inline void report(bool ok, const char* expr, const char* file, int line, const std::string& extra = "") {
  ++st().checks;
  if (ok) return;
  ++st().failures;
  std::fprintf(stderr, "  FAILED %s:%d: %s %s\n", file, line, expr, extra.c_str());
}

struct Subcase {
  bool entered = false;
  explicit Subcase(const char* name) {
    State& s = st();
    if (s.stack.size() < s.max_level) { s.reenter = true; return; }   // a subcase of this level already ran in this pass
    s.stack.push_back(name);
    if (s.passed.count(s.stack) != 0) { s.stack.pop_back(); return; }
    s.max_level = s.stack.size();
    entered = true;
  }
  ~Subcase() {
    if (!entered) return;
    State& s = st();
    if (!s.reenter) s.passed.insert(s.stack);
    s.stack.pop_back();
  }
  explicit operator bool() const { return entered; }
};

inline int run_all(int argc, char** argv) {
  std::vector<std::string> only, skip;
  for (int i = 1; i < argc; ++i) {
    if (std::strcmp(argv[i], "-x") == 0 && i + 1 < argc) skip.push_back(argv[++i]);
    else only.push_back(argv[i]);
  }
  int ran = 0, bad_cases = 0, skipped = 0;
  for (const Case& c : registry()) {
    const std::string name = c.name;
    bool take = only.empty();
    for (const auto& o : only) take = take || name.find(o) != std::string::npos;
    for (const auto& x : skip) if (name.find(x) != std::string::npos) take = false;
    if (!take) { ++skipped; continue; }
    State& s = st();
    const int before = s.failures;
    std::fprintf(stderr, "[case] %s\n", c.name);
    s.passed.clear();
    do {
      s.reenter = false; s.max_level = 0; s.stack.clear();
      try {
        c.body();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "  UNEXPECTED EXCEPTION: %s\n", e.what());
        break;
      }
    } while (s.reenter);
    ++ran;
    if (s.failures != before) ++bad_cases;
  }
  std::printf("[doctest-shim] test cases: %d | failed: %d | skipped: %d | assertions: %d | failed: %d\n", ran, bad_cases, skipped,
              st().checks, st().failures);
  return st().failures == 0 ? 0 : 1;
}

template <class E>
inline bool what_matches(const E& e, const char* substr) { return std::string(e.what()).find(substr) != std::string::npos; }
template <class E>
inline bool what_matches(const E& e, const std::string& substr) { return std::string(e.what()).find(substr) != std::string::npos; }
template <class E>
inline bool what_matches(const E& e, const Contains& c) { return std::string(e.what()).find(c.s) != std::string::npos; }

template <class... Args>
inline std::string concat(const Args&... args) {
  std::ostringstream os;
  (void)std::initializer_list<int>{((os << args), 0)...};
  return os.str();
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                                   \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                     \
  static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, DOCTEST_CAT(doctest_case_, __LINE__), __FILE__); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name})
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                              \
  do {                                                                            \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                              \
    doctest::detail::report(ok_, #__VA_ARGS__, __FILE__, __LINE__);               \
    if (!ok_) throw doctest::detail::Abort{};                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                       \
    bool thrown_ = false;                                                                    \
    try { (void)(expr); } catch (const __VA_ARGS__&) { thrown_ = true; } catch (...) {}      \
    doctest::detail::report(thrown_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__);     \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                                   \
  do {                                                                                                          \
    bool thrown_ = false;                                                                                       \
    std::string what_;                                                                                          \
    try { (void)(expr); } catch (const __VA_ARGS__& e_) { what_ = e_.what(); thrown_ = doctest::detail::what_matches(e_, with); } catch (...) {} \
    doctest::detail::report(thrown_, #expr " throws with " #with, __FILE__, __LINE__, "got: " + what_);          \
  } while (0)
#define CHECK_NOTHROW(...)                                                            \
  do {                                                                                \
    bool ok_ = true;                                                                  \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                         \
    doctest::detail::report(ok_, #__VA_ARGS__ " does not throw", __FILE__, __LINE__); \
  } while (0)
#define MESSAGE(...) std::fprintf(stderr, "  MESSAGE: %s\n", doctest::detail::concat(__VA_ARGS__).c_str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
