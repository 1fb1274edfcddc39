// TEST INFRASTRUCTURE ONLY (oracle/_ref build). A minimal stand-in for the doctest framework.
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) are written against doctest,
// which the reference vendors under proj/vendor/ (git-ignored, absent here: proj/.gitignore:2).
// This header implements the subset those files use -- TEST_CASE, TEST_SUITE_BEGIN/END, CHECK,
// CHECK_MESSAGE, CHECK_THROWS_AS, REQUIRE, FAIL, doctest::Approx and a main() honouring
// --test-suite=<name> -- so the reference's own suites run unmodified against oracle/_ref.
// doctest::Approx follows doctest's documented rule: |a - b| < eps * (scale + max(|a|, |b|)),
// default eps = 100 * FLT_EPSILON, scale 1.
#ifndef PF_SHIM_DOCTEST_H
#define PF_SHIM_DOCTEST_H

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = double(FLT_EPSILON) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct Case {
  const char* name;
  const char* suite;
  const char* file;
  int line;
  void (*fn)();
};

struct RequireFailed {};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& case_failures() {
  static int n = 0;
  return n;
}
inline long& assertions() {
  static long n = 0;
  return n;
}

inline int reg(const char* name, const char* suite, const char* file, int line, void (*fn)()) {
  registry().push_back({name, suite, file, line, fn});
  return 0;
}

template <class... T>
std::string cat(const T&... parts) {
  std::ostringstream os;
  (os << ... << parts);
  return os.str();
}

inline void fail(const char* file, int line, const std::string& what) {
  ++case_failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}

}  // namespace detail
}  // namespace doctest

// Each translation unit names its suite with TEST_SUITE_BEGIN("x") at file scope; cases that
// follow it register under that name. Before any TEST_SUITE_BEGIN the suite is "".
namespace {
[[maybe_unused]] const char* pf_doctest_suite = "";
}

#define PF_DT_CAT2(a, b) a##b
#define PF_DT_CAT(a, b) PF_DT_CAT2(a, b)

#define TEST_SUITE_BEGIN(name)                                                 \
  namespace {                                                                  \
  [[maybe_unused]] const int PF_DT_CAT(pf_dt_suite_, __LINE__) = (pf_doctest_suite = name, 0); \
  }                                                                            \
  static_assert(true, "")
#define TEST_SUITE_END() static_assert(true, "")

#define PF_DT_CASE(fn, name)                                                                    \
  static void fn();                                                                             \
  namespace {                                                                                   \
  [[maybe_unused]] const int PF_DT_CAT(fn, _reg) =                                              \
      doctest::detail::reg(name, pf_doctest_suite, __FILE__, __LINE__, &fn);                   \
  }                                                                                             \
  static void fn()
#define TEST_CASE(name) PF_DT_CASE(PF_DT_CAT(pf_dt_case_, __LINE__), name)

#define CHECK(...)                                                                  \
  do {                                                                              \
    ++doctest::detail::assertions();                                                \
    if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_MESSAGE(cond, ...)                                                          \
  do {                                                                                    \
    ++doctest::detail::assertions();                                                      \
    if (!(cond)) doctest::detail::fail(__FILE__, __LINE__, std::string("CHECK_MESSAGE(" #cond "): ") + doctest::detail::cat(__VA_ARGS__)); \
  } while (0)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    ++doctest::detail::assertions();                                                  \
    if (!(__VA_ARGS__)) {                                                             \
      doctest::detail::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");         \
      throw doctest::detail::RequireFailed{};                                         \
    }                                                                                 \
  } while (0)
#define FAIL(msg)                                                                   \
  do {                                                                              \
    doctest::detail::fail(__FILE__, __LINE__, std::string("FAIL: ") + std::string(msg)); \
    throw doctest::detail::RequireFailed{};                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    ++doctest::detail::assertions();                                                      \
    bool pf_dt_ok = false;                                                                \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      pf_dt_ok = true;                                                                    \
    } catch (...) {                                                                       \
    }                                                                                     \
    if (!pf_dt_ok) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::string suite;
  bool any_suite = true;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--test-suite=", 13) == 0) {
      suite = argv[i] + 13;
      any_suite = false;
    }
  }
  int cases = 0, failed_cases = 0;
  for (const auto& c : doctest::detail::registry()) {
    if (!any_suite && suite != c.suite) continue;
    ++cases;
    int before = doctest::detail::case_failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest::detail::fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      doctest::detail::fail(c.file, c.line, "unexpected exception");
    }
    if (doctest::detail::case_failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE(\"%s\") [%s]\n", c.name, c.suite);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | failed: %d\n",
              cases, cases - failed_cases, failed_cases, doctest::detail::assertions(),
              doctest::detail::case_failures());
  return failed_cases == 0 && cases > 0 ? 0 : 1;
}
#endif

#endif  // PF_SHIM_DOCTEST_H
