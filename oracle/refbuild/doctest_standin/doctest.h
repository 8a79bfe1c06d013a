// doctest.h STAND-IN — TEST INFRASTRUCTURE ONLY (oracle/refbuild).
//
// The reference's unit tests (proj/tests/test_*.cpp) are written against
// doctest, which the reference does not commit (proj/README.md:41-43) and this
// image does not have.  This is our own minimal runner for exactly the macros
// those files use — TEST_CASE, SUBCASE (each leaf re-runs the test case from
// the top, like doctest), CHECK / CHECK_FALSE / REQUIRE, CHECK_NOTHROW,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CAPTURE, FAIL, doctest::Approx — so
// that the UNMODIFIED test sources compile where they lie and run against the
// reference build (oracle/refbuild/Makefile, target tests).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double value, eps = static_cast<double>(FLT_EPSILON) * 100.0, scale_ = 1.0;
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - value) < eps * (scale_ + std::fmax(std::fabs(x), std::fabs(value)));
  }
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& b, double a) { return b.matches(a); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& b, double a) { return !b.matches(a); }
inline bool operator<=(double a, const Approx& b) { return a < b.value || b.matches(a); }
inline bool operator>=(double a, const Approx& b) { return a > b.value || b.matches(a); }

namespace mini {

struct AbortTest {};

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { cases().push_back({name, fn}); }
};

struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  // SUBCASE bookkeeping for one pass over a test case: `path` is the chosen
  // child index at each nesting depth; a pass enters, at each depth, only the
  // child numbered path[depth], and records how many siblings it saw.
  std::vector<int> path, seen;
  int depth = 0;
  bool more = false;
};
inline State& state() {
  static State s;
  return s;
}

inline void fail(const char* file, int line, const char* what, const std::string& extra = "") {
  State& s = state();
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: FAILED: %s %s\n", file, line, what, extra.c_str());
}
inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
  ++state().checks;
  if (ok) return;
  fail(file, line, expr);
  if (require) throw AbortTest{};
}

// RAII guard of one SUBCASE block.
struct Subcase {
  bool entered = false;
  explicit Subcase(const char*) {
    State& s = state();
    const int d = s.depth;
    if (static_cast<int>(s.seen.size()) <= d) s.seen.resize(static_cast<std::size_t>(d) + 1, 0);
    if (static_cast<int>(s.path.size()) <= d) s.path.resize(static_cast<std::size_t>(d) + 1, 0);
    const int index = s.seen[static_cast<std::size_t>(d)]++;
    if (index == s.path[static_cast<std::size_t>(d)]) {
      entered = true;
      ++s.depth;
      if (static_cast<int>(s.seen.size()) > s.depth) s.seen[static_cast<std::size_t>(s.depth)] = 0;
    }
  }
  ~Subcase() {
    if (entered) --state().depth;
  }
  explicit operator bool() const { return entered; }
};

// Advances `path` to the next leaf (depth-first); false when all were run.
inline bool next_path() {
  State& s = state();
  for (int d = static_cast<int>(s.seen.size()) - 1; d >= 0; --d) {
    if (static_cast<int>(s.path.size()) <= d) s.path.resize(static_cast<std::size_t>(d) + 1, 0);
    if (s.path[static_cast<std::size_t>(d)] + 1 < s.seen[static_cast<std::size_t>(d)]) {
      ++s.path[static_cast<std::size_t>(d)];
      s.path.resize(static_cast<std::size_t>(d) + 1);
      return true;
    }
  }
  return false;
}

inline int run_all() {
  State& s = state();
  int failed_cases = 0, runs = 0;
  for (const Case& c : cases()) {
    s.path.clear();
    bool case_failed = false;
    for (;;) {
      s.seen.assign(s.path.size() + 1, 0);
      s.depth = 0;
      s.case_failed = false;
      ++runs;
      try {
        c.fn();
      } catch (const AbortTest&) {
      } catch (const std::exception& e) {
        fail(c.name, 0, "unexpected exception:", e.what());
      } catch (...) {
        fail(c.name, 0, "unexpected exception of unknown type");
      }
      case_failed = case_failed || s.case_failed;
      // keep only depths that exist on the path just taken
      std::vector<int> seen = s.seen;
      s.seen = seen;
      if (!next_path()) break;
    }
    if (case_failed) {
      ++failed_cases;
      std::printf("TEST CASE FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest stand-in] test cases: %zu | %zu passed | %d failed\n", cases().size(),
              cases().size() - static_cast<std::size_t>(failed_cases), failed_cases);
  std::printf("[doctest stand-in] assertions: %ld | %ld passed | %ld failed | passes over cases: %d\n",
              s.checks, s.checks - s.failed_checks, s.failed_checks, runs);
  return failed_cases == 0 && s.failed_checks == 0 ? 0 : 1;
}

}  // namespace mini
}  // namespace doctest

#define DOCTEST_MINI_CAT2(a, b) a##b
#define DOCTEST_MINI_CAT(a, b) DOCTEST_MINI_CAT2(a, b)

#define TEST_CASE(name)                                                                   \
  static void DOCTEST_MINI_CAT(doctest_mini_case_, __LINE__)();                            \
  static ::doctest::mini::Registrar DOCTEST_MINI_CAT(doctest_mini_reg_, __LINE__)(         \
      name, &DOCTEST_MINI_CAT(doctest_mini_case_, __LINE__));                              \
  static void DOCTEST_MINI_CAT(doctest_mini_case_, __LINE__)()

#define SUBCASE(name) \
  if (::doctest::mini::Subcase DOCTEST_MINI_CAT(doctest_mini_sub_, __LINE__){name})

#define CHECK(...) ::doctest::mini::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")", false)
#define CHECK_FALSE(...) ::doctest::mini::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::mini::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")", true)
#define CAPTURE(...) ((void)0)
#define INFO(...) ((void)0)
#define FAIL(...)                                                          \
  do {                                                                     \
    ::doctest::mini::fail(__FILE__, __LINE__, "FAIL(" #__VA_ARGS__ ")");   \
    throw ::doctest::mini::AbortTest{};                                    \
  } while (0)

#define CHECK_NOTHROW(...)                                                                  \
  do {                                                                                      \
    ++::doctest::mini::state().checks;                                                      \
    try {                                                                                   \
      __VA_ARGS__;                                                                          \
    } catch (...) {                                                                         \
      ::doctest::mini::fail(__FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ") threw");   \
    }                                                                                       \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                       \
    ++::doctest::mini::state().checks;                                                       \
    bool doctest_mini_ok = false;                                                            \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const std::remove_reference<__VA_ARGS__>::type&) {                              \
      doctest_mini_ok = true;                                                                \
    } catch (...) {                                                                          \
    }                                                                                        \
    if (!doctest_mini_ok)                                                                    \
      ::doctest::mini::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                \
  do {                                                                                       \
    ++::doctest::mini::state().checks;                                                       \
    bool doctest_mini_ok = false;                                                            \
    std::string doctest_mini_msg;                                                            \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const std::remove_reference<__VA_ARGS__>::type& e) {                            \
      doctest_mini_msg = e.what();                                                           \
      doctest_mini_ok = doctest_mini_msg == std::string(with);                               \
    } catch (...) {                                                                          \
    }                                                                                        \
    if (!doctest_mini_ok)                                                                    \
      ::doctest::mini::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ", " #with ")", \
                            "got: " + doctest_mini_msg);                                     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::mini::run_all(); }
#endif
