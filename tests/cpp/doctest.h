// doctest.h -- minimal stand-in for the doctest macros the reference's hot-path unit tests use
// (TEST_CASE, SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS), so those test files compile
// unchanged against the B200 host API.  Test infrastructure only.
//
// SUBCASE follows doctest's rule for flat subcases: the test body runs once per subcase,
// executing the shared code plus exactly one subcase each pass.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {

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
  long checks = 0, failed = 0;
  int target = 0, seen = 0;
  bool case_failed = false;
};
inline State& st() {
  static State s;
  return s;
}

struct Abort {};

inline bool reg(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return true;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++st().checks;
  if (ok) return;
  ++st().failed;
  st().case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

inline bool enter_subcase() { return st().seen++ == st().target; }

inline int run_all(int argc, char** argv) {
  int cases = 0, bad = 0;
  for (const Case& c : registry()) {
    if (argc > 1) {  // optional substring filter on the test name
      bool hit = false;
      for (int i = 1; i < argc; ++i) hit |= std::string(c.name).find(argv[i]) != std::string::npos;
      if (!hit) continue;
    }
    ++cases;
    st().case_failed = false;
    for (st().target = 0;; ++st().target) {
      st().seen = 0;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        ++st().failed;
        st().case_failed = true;
        std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name,
                     e.what());
      }
      if (st().seen <= st().target + 1) break;  // no further subcases
    }
    bad += st().case_failed;
    std::printf("[%s] %s\n", st().case_failed ? "FAIL" : "PASS", c.name);
  }
  std::printf("test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n", cases,
              cases - bad, bad, st().checks, st().failed);
  return bad ? 1 : 0;
}

}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define TEST_CASE(name)                                                                        \
  static void DS_CAT(ds_case_, __LINE__)();                                                    \
  static const bool DS_CAT(ds_reg_, __LINE__) =                                                \
      doctest_shim::reg(name, __FILE__, __LINE__, &DS_CAT(ds_case_, __LINE__));                \
  static void DS_CAT(ds_case_, __LINE__)()
#define SUBCASE(name) if (doctest_shim::enter_subcase())
#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                           \
  do {                                                                                         \
    const bool ds_ok = static_cast<bool>(__VA_ARGS__);                                         \
    doctest_shim::report(ds_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                  \
    if (!ds_ok) throw doctest_shim::Abort{};                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                             \
  do {                                                                                         \
    bool ds_ok = false;                                                                        \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const __VA_ARGS__&) {                                                             \
      ds_ok = true;                                                                            \
    } catch (...) {                                                                            \
    }                                                                                          \
    doctest_shim::report(ds_ok, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);                 \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest_shim::run_all(argc, argv); }
#endif
