// TEST INFRASTRUCTURE ONLY (oracle/): a small stand-in for the part of
// doctest the reference's tests (proj/tests/*.cpp) use -- TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so those files compile unmodified in
// this image, which has no doctest.h. Written from the macro
// names only. The runner prints one line per failed check and per test case,
// takes an optional substring filter (argv[1], or "-x<substring>" to
// exclude; several allowed), and returns the number of failed cases.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct State {
  int checks = 0, failed_checks = 0;
  int case_failed = 0;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().checks;
  if (ok) return;
  ++state().failed_checks;
  ++state().case_failed;
  if (state().case_failed <= 10)
    std::printf("  %s:%d: %s( %s ) failed\n", file, line, kind, expr);
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - v_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(v_)));
  }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-5;  // float epsilon * 100
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }


inline int run(int argc, char** argv) {
  int failed = 0, ran = 0;
  for (const TestCase& t : registry()) {
    bool take = true, any_include = false, included = false;
    for (int i = 1; i < argc; ++i) {
      if (std::strncmp(argv[i], "-x", 2) == 0) {
        if (std::strstr(t.name, argv[i] + 2)) take = false;
      } else {
        any_include = true;
        if (std::strstr(t.name, argv[i])) included = true;
      }
    }
    if (!take || (any_include && !included)) continue;
    ++ran;
    state().case_failed = 0;
    try {
      t.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++state().case_failed;
      std::printf("  %s:%d: unexpected exception: %s\n", t.file, t.line, e.what());
    } catch (...) {
      ++state().case_failed;
      std::printf("  %s:%d: unexpected exception\n", t.file, t.line);
    }
    std::printf("[%s] %s\n", state().case_failed ? "FAILED" : "  ok  ", t.name);
    std::fflush(stdout);
    if (state().case_failed) ++failed;
  }
  std::printf("test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", ran,
              ran - failed, failed, state().checks, state().failed_checks);
  return failed;
}

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                              \
  static void fn();                                                                    \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                                   \
    doctest::report(doctest_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                 \
    if (!doctest_ok) throw doctest::RequireFailed{};                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool doctest_thrown = false;                                                              \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const __VA_ARGS__&) {                                                            \
      doctest_thrown = true;                                                                  \
    } catch (...) {                                                                           \
    }                                                                                         \
    doctest::report(doctest_thrown, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                    \
  do {                                                                                        \
    bool doctest_ok = true;                                                                   \
    try {                                                                                     \
      static_cast<void>(__VA_ARGS__);                                                         \
    } catch (...) {                                                                           \
      doctest_ok = false;                                                                     \
    }                                                                                         \
    doctest::report(doctest_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);           \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run(argc, argv) ? 1 : 0; }
#endif
