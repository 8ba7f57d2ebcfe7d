// Minimal doctest-compatible test harness — TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) use doctest from a gitignored
// vendor/ tree (proj/.gitignore:2) that is absent here.  This header provides the subset they use,
// with doctest's documented semantics: TEST_CASE registration, CHECK / REQUIRE / CHECK_THROWS_AS,
// and doctest::Approx (default epsilon = 100 * FLT_EPSILON, scale 1:
// |a - b| < eps * (scale + max(|a|, |b|))).  DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN provides main(),
// which accepts doctest's --test-case=<a,b> / --test-case-exclude=<a,b> filters (exact names or
// '*' suffix wildcards) and prints a doctest-style summary.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

namespace detail {
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
struct RequireFailed {};
struct Counters {
  long asserts = 0, failed_asserts = 0;
  bool current_failed = false;
  const char* current = "";
};
inline Counters& counters() {
  static Counters c;
  return c;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  Counters& c = counters();
  ++c.asserts;
  if (!ok) {
    ++c.failed_asserts;
    c.current_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!  [test case: %s]\n", file, line, kind, expr,
                 c.current);
  }
}
inline bool name_matches(const std::string& pat, const std::string& name) {
  if (!pat.empty() && pat.back() == '*') return name.compare(0, pat.size() - 1, pat, 0, pat.size() - 1) == 0;
  return pat == name;
}
inline std::vector<std::string> split_list(const std::string& s) {
  std::vector<std::string> out;
  size_t a = 0;
  while (a <= s.size()) {
    size_t b = s.find(',', a);
    if (b == std::string::npos) b = s.size();
    if (b > a) out.push_back(s.substr(a, b - a));
    a = b + 1;
  }
  return out;
}
inline int run(int argc, char** argv) {
  std::vector<std::string> include, exclude;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto val = [&](const char* key) -> const char* {
      const size_t n = std::strlen(key);
      return a.compare(0, n, key) == 0 ? argv[i] + n : nullptr;
    };
    if (const char* v = val("--test-case=")) include = split_list(v);
    if (const char* v = val("-tc=")) include = split_list(v);
    if (const char* v = val("--test-case-exclude=")) exclude = split_list(v);
    if (const char* v = val("-tce=")) exclude = split_list(v);
  }
  long run_cases = 0, failed_cases = 0, skipped = 0;
  for (const TestCase& tc : registry()) {
    bool take = include.empty();
    for (auto& p : include) take = take || name_matches(p, tc.name);
    for (auto& p : exclude) take = take && !name_matches(p, tc.name);
    if (!take) {
      ++skipped;
      continue;
    }
    Counters& c = counters();
    c.current = tc.name;
    c.current_failed = false;
    ++run_cases;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      c.current_failed = true;
      std::fprintf(stderr, "%s:%d: ERROR: test case THREW exception: %s  [test case: %s]\n", tc.file, tc.line,
                   e.what(), tc.name);
    } catch (...) {
      c.current_failed = true;
      std::fprintf(stderr, "%s:%d: ERROR: test case THREW an unknown exception  [test case: %s]\n", tc.file,
                   tc.line, tc.name);
    }
    if (c.current_failed) ++failed_cases;
  }
  const Counters& c = counters();
  std::printf("[doctest] test cases: %ld | %ld passed | %ld failed | %ld skipped\n", run_cases,
              run_cases - failed_cases, failed_cases, skipped);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed |\n", c.asserts, c.asserts - c.failed_asserts,
              c.failed_asserts);
  std::printf("[doctest] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
  return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                           \
  static void fn();                                                                                \
  static const ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_anon_func_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                    \
  do {                                                                                                  \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                           \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);               \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                        \
  } while (0)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, ...)                                                                      \
  do {                                                                                                  \
    bool doctest_ok_ = false;                                                                           \
    try {                                                                                               \
      static_cast<void>(expr);                                                                          \
    } catch (const __VA_ARGS__&) {                                                                      \
      doctest_ok_ = true;                                                                               \
    } catch (...) {                                                                                     \
    }                                                                                                   \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                  \
  do {                                                                                       \
    bool doctest_ok_ = true;                                                                 \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (...) {                                                                          \
      doctest_ok_ = false;                                                                   \
    }                                                                                        \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
