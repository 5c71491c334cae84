// TEST INFRASTRUCTURE ONLY.  A minimal doctest-compatible shim (doctest itself
// is git-ignored/absent in the reference, proj/.gitignore:2) so the reference's
// own unit tests (/root/reference/proj/tests/*.cpp) can run against the
// oracle/_ref build and pin it.  Supports exactly the macros those tests use:
// TEST_CASE, CHECK, CHECK_MESSAGE, CHECK_THROWS_AS, REQUIRE, REQUIRE_MESSAGE.
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
struct Registrar {
  Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};
inline int& checks() { static int c = 0; return c; }
inline int& failures() { static int c = 0; return c; }
inline bool& case_failed() { static bool b = false; return b; }
inline void fail(const char* file, int line, const char* expr, const std::string& msg = "") {
  failures()++;
  case_failed() = true;
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s %s\n", file, line, expr, msg.c_str());
}
inline std::string to_msg(const char* s) { return s ? s : ""; }
inline std::string to_msg(const std::string& s) { return s; }
}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define TEST_CASE(name)                                                                 \
  static void DS_CAT(ds_case_, __LINE__)();                                             \
  static doctest_shim::Registrar DS_CAT(ds_reg_, __LINE__)(name, __FILE__, __LINE__,    \
                                                           &DS_CAT(ds_case_, __LINE__)); \
  static void DS_CAT(ds_case_, __LINE__)()

#define CHECK(...)                                                                    \
  do {                                                                                \
    doctest_shim::checks()++;                                                         \
    if (!(__VA_ARGS__)) doctest_shim::fail(__FILE__, __LINE__, #__VA_ARGS__);         \
  } while (0)
#define CHECK_MESSAGE(cond, msg)                                                      \
  do {                                                                                \
    doctest_shim::checks()++;                                                         \
    if (!(cond)) doctest_shim::fail(__FILE__, __LINE__, #cond, doctest_shim::to_msg(msg)); \
  } while (0)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    doctest_shim::checks()++;                                                         \
    if (!(__VA_ARGS__)) {                                                             \
      doctest_shim::fail(__FILE__, __LINE__, #__VA_ARGS__);                           \
      throw doctest_shim::RequireFailed{};                                            \
    }                                                                                 \
  } while (0)
#define REQUIRE_MESSAGE(cond, msg)                                                    \
  do {                                                                                \
    doctest_shim::checks()++;                                                         \
    if (!(cond)) {                                                                    \
      doctest_shim::fail(__FILE__, __LINE__, #cond, doctest_shim::to_msg(msg));       \
      throw doctest_shim::RequireFailed{};                                            \
    }                                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, ex)                                                     \
  do {                                                                                \
    doctest_shim::checks()++;                                                         \
    bool ds_ok = false;                                                               \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const ex&) {                                                             \
      ds_ok = true;                                                                   \
    } catch (...) {                                                                   \
    }                                                                                 \
    if (!ds_ok) doctest_shim::fail(__FILE__, __LINE__, #expr " throws " #ex);         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : doctest_shim::registry()) {
    doctest_shim::case_failed() = false;
    try {
      c.fn();
    } catch (const doctest_shim::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest_shim::fail(c.file, c.line, "unexpected exception", e.what());
    }
    if (doctest_shim::case_failed()) {
      failed_cases++;
      std::fprintf(stderr, "FAILED CASE: %s (%s:%d)\n", c.name, c.file, c.line);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %d | failed checks: %d\n",
              doctest_shim::registry().size(), failed_cases, doctest_shim::checks(),
              doctest_shim::failures());
  return failed_cases ? 1 : 0;
}
#endif
