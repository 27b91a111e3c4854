// TEST INFRASTRUCTURE ONLY -- a minimal stand-in for the doctest single
// header the reference's unit tests include (proj/tests/*.cpp; the vendored
// header is absent from /root/reference).  It implements only
// what those files use: TEST_CASE, flat SUBCASE (each test case re-runs once
// per subcase, entering exactly one, as doctest does), CHECK, CHECK_FALSE,
// REQUIRE, FAIL, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS and the
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN entry point.  Failures print file:line
// and the expression; the process exits nonzero when any check failed.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {

struct Case {
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct State {
  int failures = 0, checks = 0;
  int target = 0, seen = 0;  // subcase to enter in this pass / subcases met so far
  const char* current = "";
};

inline State& st() {
  static State s;
  return s;
}

struct Abort {};

inline void fail(const char* file, int line, const char* what) {
  ++st().failures;
  std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, st().current, what);
}

inline void check(bool ok, const char* file, int line, const char* what, bool require) {
  ++st().checks;
  if (ok) return;
  fail(file, line, what);
  if (require) throw Abort{};
}

inline bool enter_subcase() { return st().seen++ == st().target; }

struct Reg {
  Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

inline int run_all() {
  int cases = 0;
  for (const Case& c : registry()) {
    st().current = c.name;
    for (int target = 0;; ++target) {
      st().target = target;
      st().seen = 0;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        fail("<test case>", 0, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        fail("<test case>", 0, "unexpected exception");
      }
      if (st().seen <= target + 1) break;  // no further subcase to enter
    }
    ++cases;
  }
  std::printf("[doctest shim] %d test cases, %d checks, %d failed\n", cases, st().checks, st().failures);
  return st().failures ? 1 : 0;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST(fn, name)                                        \
  static void fn();                                                        \
  static doctest_shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, &fn);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)
#define SUBCASE(name) if (doctest_shim::enter_subcase())
#define CHECK(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) doctest_shim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define FAIL(msg)                                   \
  do {                                              \
    doctest_shim::fail(__FILE__, __LINE__, "FAIL"); \
    throw doctest_shim::Abort{};                    \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool doctest_shim_ok = false;                                                        \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const __VA_ARGS__&) {                                                       \
      doctest_shim_ok = true;                                                            \
    } catch (...) {                                                                      \
    }                                                                                    \
    doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, #expr " throws " #__VA_ARGS__, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                             \
  do {                                                                                   \
    bool doctest_shim_ok = false;                                                        \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const __VA_ARGS__& e) {                                                     \
      doctest_shim_ok = std::string(e.what()) == std::string(msg);                       \
    } catch (...) {                                                                      \
    }                                                                                    \
    doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, #expr " throws " #__VA_ARGS__ " with " #msg, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
