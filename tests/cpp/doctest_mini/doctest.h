// doctest.h -- a minimal stand-in for the doctest macros the reference's unit
// tests use (TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW), written for this repo so those test files compile UNCHANGED
// against include/densegraph/*.hpp and run on the device (oracle/Makefile
// target ref-tests; tests/test_gpu_parity.py).  TEST INFRASTRUCTURE ONLY.
//
// SUBCASE semantics follow doctest: a test case is re-run once per leaf
// subcase, entering exactly one subcase per nesting level on each run.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace dmini {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct State {
  std::vector<int> path;    // subcase index to enter at each depth
  std::vector<int> counts;  // subcases seen at each depth in this run
  int depth = 0;
  long checks = 0, failures = 0;
  const char* current = "";
};

inline State& state() {
  static State s;
  return s;
}

struct Abort {};  // a failed REQUIRE ends the current run of the test case

inline void fail(const char* file, int line, const char* what) {
  State& s = state();
  ++s.failures;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.current, what);
}

inline bool check(bool ok, const char* file, int line, const char* what) {
  ++state().checks;
  if (!ok) fail(file, line, what);
  return ok;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct Subcase {
  bool entered = false;
  explicit Subcase(const char*) {
    State& s = state();
    const int d = s.depth;
    if ((int)s.counts.size() <= d) s.counts.resize(d + 1, 0);
    const int idx = s.counts[d]++;
    if ((int)s.path.size() > d) {
      entered = idx == s.path[d];
    } else if (idx == 0) {
      entered = true;
      s.path.push_back(0);
    }
    if (entered) {
      ++s.depth;
      if ((int)s.counts.size() > s.depth) s.counts[s.depth] = 0;
    }
  }
  ~Subcase() {
    if (entered) --state().depth;
  }
  explicit operator bool() const { return entered; }
};

inline int run_all() {
  State& s = state();
  long cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    s.current = c.name;
    s.path.clear();
    const long f0 = s.failures;
    for (;;) {
      s.counts.assign(1, 0);
      s.depth = 0;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        fail(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        fail(c.file, c.line, "unexpected exception");
      }
      // next leaf: the deepest level with an unvisited sibling
      int d = (int)s.path.size() - 1;
      while (d >= 0 && !((int)s.counts.size() > d && s.counts[d] > s.path[d] + 1)) --d;
      if (d < 0) break;
      ++s.path[d];
      s.path.resize(d + 1);
    }
    ++cases;
    if (s.failures != f0) ++failed_cases;
  }
  std::printf("[doctest-mini] test cases: %ld | %ld passed | %ld failed; assertions: %ld, failures: %ld\n",
              cases, cases - failed_cases, failed_cases, s.checks, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace dmini

#define DMINI_CAT_(a, b) a##b
#define DMINI_CAT(a, b) DMINI_CAT_(a, b)
#define TEST_CASE(name)                                                                 \
  static void DMINI_CAT(dmini_case_, __LINE__)();                                       \
  static ::dmini::Registrar DMINI_CAT(dmini_reg_, __LINE__)(name, __FILE__, __LINE__,   \
                                                            &DMINI_CAT(dmini_case_, __LINE__)); \
  static void DMINI_CAT(dmini_case_, __LINE__)()
#define SUBCASE(name) if (const ::dmini::Subcase DMINI_CAT(dmini_sc_, __LINE__){name})
#define CHECK(...) ::dmini::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) \
  ::dmini::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "not " #__VA_ARGS__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    if (!::dmini::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__))   \
      throw ::dmini::Abort{};                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                      \
  do {                                                                                   \
    bool dmini_ok_ = false;                                                              \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const type&) {                                                              \
      dmini_ok_ = true;                                                                  \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::dmini::check(dmini_ok_, __FILE__, __LINE__, #expr " throws " #type);              \
  } while (0)
#define CHECK_NOTHROW(expr)                                                              \
  do {                                                                                   \
    bool dmini_ok_ = true;                                                               \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (...) {                                                                      \
      dmini_ok_ = false;                                                                 \
    }                                                                                    \
    ::dmini::check(dmini_ok_, __FILE__, __LINE__, #expr " does not throw");             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::dmini::run_all(); }
#endif
