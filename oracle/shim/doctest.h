// TEST INFRASTRUCTURE ONLY (oracle build shim).
//
// Minimal stand-in for the doctest single header the reference tests expect
// under proj/vendor/ (absent; proj/.gitignore:2).  Supports exactly the macros
// the reference tests use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, with a main() under DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Command line: -tc=<substr>[,<substr>...] selects cases, -tce=<substr>
// excludes cases (substring match on the case name; '*' characters ignored).
#ifndef CTG_ORACLE_SHIM_DOCTEST_H
#define CTG_ORACLE_SHIM_DOCTEST_H

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace ctg_doctest {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Stats {
  long checks = 0, failed_checks = 0;
};
inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailed {};

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed_checks;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, fatal ? "REQUIRE" : "CHECK", expr);
  if (fatal) throw RequireFailed{};
}

inline std::vector<std::string> split(const char* s) {
  std::vector<std::string> out;
  std::string cur;
  for (const char* p = s; *p; ++p) {
    if (*p == ',') {
      out.push_back(cur);
      cur.clear();
    } else if (*p != '*') {
      cur += *p;
    }
  }
  out.push_back(cur);
  return out;
}

inline bool matches(const std::string& name, const std::vector<std::string>& pats) {
  for (const auto& p : pats)
    if (!p.empty() && name.find(p) != std::string::npos) return true;
  return false;
}

inline int run(int argc, char** argv) {
  std::vector<std::string> inc, exc;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) inc = split(argv[i] + 4);
    if (std::strncmp(argv[i], "-tce=", 5) == 0) exc = split(argv[i] + 5);
  }
  int cases = 0, failed_cases = 0;
  for (const auto& c : registry()) {
    std::string name(c.name);
    if (!inc.empty() && !matches(name, inc)) continue;
    if (!exc.empty() && matches(name, exc)) continue;
    ++cases;
    long before = stats().failed_checks;
    bool ok = true;
    auto t0 = std::chrono::steady_clock::now();
    try {
      c.fn();
    } catch (const RequireFailed&) {
      ok = false;
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
      ++stats().failed_checks;
      ok = false;
    }
    double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats().failed_checks != before) ok = false;
    if (!ok) ++failed_cases;
    std::fprintf(stderr, "[%s] %s (%.3fs)\n", ok ? "PASS" : "FAIL", c.name, sec);
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases,
              failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
              stats().checks - stats().failed_checks, stats().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace ctg_doctest

#define CTG_DT_CAT2(a, b) a##b
#define CTG_DT_CAT(a, b) CTG_DT_CAT2(a, b)
#define TEST_CASE(name)                                                                 \
  static void CTG_DT_CAT(ctg_dt_fn_, __LINE__)();                                      \
  static ctg_doctest::Registrar CTG_DT_CAT(ctg_dt_reg_, __LINE__)(                      \
      name, &CTG_DT_CAT(ctg_dt_fn_, __LINE__), __FILE__, __LINE__);                     \
  static void CTG_DT_CAT(ctg_dt_fn_, __LINE__)()

#define CHECK(...) ctg_doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ctg_doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) ctg_doctest::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_THROWS_AS(expr, exc)                                          \
  do {                                                                      \
    bool ctg_dt_ok = false;                                                 \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const exc&) {                                                  \
      ctg_dt_ok = true;                                                     \
    } catch (...) {                                                         \
    }                                                                       \
    ctg_doctest::report(ctg_dt_ok, #expr " throws " #exc, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(...)                                                  \
  do {                                                                      \
    bool ctg_dt_ok = true;                                                  \
    try {                                                                   \
      (void)(__VA_ARGS__);                                                  \
    } catch (...) {                                                         \
      ctg_dt_ok = false;                                                    \
    }                                                                       \
    ctg_doctest::report(ctg_dt_ok, #__VA_ARGS__ " nothrow", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ctg_doctest::run(argc, argv); }
#endif

#endif  // CTG_ORACLE_SHIM_DOCTEST_H
