// tests/cpp/doctest.h -- a small doctest-compatible test runner (TEST
// INFRASTRUCTURE; written for this repository, not the doctest library).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// <doctest.h>, whose vendored copy is not shipped (proj/.gitignore:2).  This
// header implements the subset those files use -- TEST_CASE, SUBCASE (doctest
// semantics: the test case body re-runs once per leaf subcase), CHECK,
// REQUIRE, CHECK_THROWS_AS, FAIL, CAPTURE and doctest::Approx -- so the
// unmodified test sources compile against include/folp and link against
// libfolp_b200.so (tests/cpp/Makefile; run by tests/test_cpp_dropin.py).
//
// Approx follows doctest's documented comparison:
//   |a - b| < eps * (scale + max(|a|, |b|)),  eps = 100 * FLT_EPSILON, scale 1.
#ifndef FOLP_TESTS_DOCTEST_SHIM_H_
#define FOLP_TESTS_DOCTEST_SHIM_H_

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool matches(double other) const {
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
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
  static std::vector<TestCase> cases;
  return cases;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

// Thrown by REQUIRE / FAIL to abandon the current run of a test case.
struct Abort {};

// Per-test-case state: which subcase paths are finished, and the path and
// bookkeeping of the current run.
struct Runner {
  std::set<std::vector<std::string>> done;
  std::vector<std::string> path;
  std::vector<bool> entered;  // a subcase was entered at depth d in this run
  std::vector<bool> pending;  // scope at depth d still has unvisited subcases
  std::vector<std::string> captures;
  long checks = 0;
  long failed_checks = 0;
  const TestCase* current = nullptr;
};

inline Runner& runner() {
  static Runner r;
  return r;
}

inline std::string path_string() {
  std::string s;
  for (const auto& p : runner().path) s += " / " + p;
  return s;
}

inline void report_failure(const char* file, int line, const std::string& what) {
  Runner& r = runner();
  ++r.failed_checks;
  std::fprintf(stderr, "%s:%d: FAILED in TEST_CASE(\"%s\")%s: %s\n", file, line,
               r.current ? r.current->name : "?", path_string().c_str(), what.c_str());
  for (const auto& c : r.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

inline bool check(bool ok, const char* file, int line, const char* macro, const char* expr) {
  ++runner().checks;
  if (!ok) report_failure(file, line, std::string(macro) + "( " + expr + " ) is false");
  return ok;
}

class Subcase {
 public:
  Subcase(const char* name) {
    Runner& r = runner();
    const size_t d = r.path.size();
    if (r.entered.size() <= d) r.entered.resize(d + 1, false);
    if (r.pending.size() <= d) r.pending.resize(d + 1, false);
    std::vector<std::string> key = r.path;
    key.emplace_back(name);
    if (r.done.count(key)) return;
    if (r.entered[d]) {  // a sibling ran in this pass: come back for this one
      for (size_t k = 0; k <= d; ++k) r.pending[k] = true;
      return;
    }
    r.entered[d] = true;
    r.path.push_back(key.back());
    r.entered.resize(d + 2, false);
    r.entered[d + 1] = false;
    r.pending.resize(d + 2, false);
    r.pending[d + 1] = false;
    active_ = true;
  }
  ~Subcase() {
    if (!active_) return;
    Runner& r = runner();
    const size_t d = r.path.size();  // depth of this subcase's own scope
    if (!r.pending[d]) r.done.insert(r.path);
    r.path.pop_back();
  }
  explicit operator bool() const { return active_; }

 private:
  bool active_ = false;
};

struct Capture {
  explicit Capture(std::string s) { runner().captures.push_back(std::move(s)); }
  ~Capture() { runner().captures.pop_back(); }
};

template <class T>
std::string to_text(const T& v) {
  std::ostringstream os;
  if constexpr (requires { os << v; }) {
    os << v;
  } else {
    os << "{?}";
  }
  return os.str();
}

}  // namespace detail

// Runs every registered test case (optionally only names containing
// `filter`, defined in a file whose path contains `file_filter`, and not
// named with `exclude`), printing one line per case; returns the number of failed cases.
inline int run_all(const char* filter, const char* file_filter, const char* exclude) {
  using namespace detail;
  int failed_cases = 0, cases = 0;
  long total_checks = 0, total_failed = 0;
  for (const TestCase& tc : registry()) {
    if (filter && *filter && !std::strstr(tc.name, filter)) continue;
    if (file_filter && *file_filter && !std::strstr(tc.file, file_filter)) continue;
    if (exclude && *exclude && std::strstr(tc.name, exclude)) continue;
    ++cases;
    Runner& r = runner();
    r = Runner{};
    r.current = &tc;
    bool ok = true;
    for (int pass = 0; pass < 10000; ++pass) {
      r.path.clear();
      r.entered.assign(1, false);
      r.pending.assign(1, false);
      r.captures.clear();
      const long before = r.failed_checks;
      try {
        tc.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        report_failure(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report_failure(tc.file, tc.line, "unexpected non-standard exception");
      }
      while (!r.path.empty()) r.path.pop_back();
      if (r.failed_checks != before) ok = false;
      if (!r.pending[0]) break;
    }
    total_checks += r.checks;
    total_failed += r.failed_checks;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s (%ld checks)\n", ok ? "PASS" : "FAIL", tc.name, r.checks);
    std::fflush(stdout);
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | checks: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, total_checks, total_failed);
  return failed_cases;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(name) DOCTEST_CAT(name, __LINE__)

#define TEST_CASE(name)                                                         \
  static void DOCTEST_UNIQUE(doctest_case_fn_)();                               \
  static const ::doctest::detail::Registrar DOCTEST_UNIQUE(doctest_case_reg_)(  \
      name, __FILE__, __LINE__, &DOCTEST_UNIQUE(doctest_case_fn_));             \
  static void DOCTEST_UNIQUE(doctest_case_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_UNIQUE(doctest_sub_){name})

#define CHECK(...) \
  ((void)::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__))
#define CHECK_FALSE(...) \
  ((void)::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__))
#define REQUIRE(...)                                                                            \
  do {                                                                                          \
    if (!::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", \
                                  #__VA_ARGS__))                                                \
      throw ::doctest::detail::Abort{};                                                         \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))

#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool doctest_threw_ = false;                                                              \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const __VA_ARGS__&) {                                                            \
      doctest_threw_ = true;                                                                  \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::detail::check(doctest_threw_, __FILE__, __LINE__, "CHECK_THROWS_AS",           \
                             #expr " throws " #__VA_ARGS__);                                  \
  } while (0)
#define CHECK_THROWS(expr)                                                                      \
  do {                                                                                          \
    bool doctest_threw_ = false;                                                                \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (...) {                                                                             \
      doctest_threw_ = true;                                                                    \
    }                                                                                           \
    ::doctest::detail::check(doctest_threw_, __FILE__, __LINE__, "CHECK_THROWS", #expr " throws"); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                    \
  do {                                                                                         \
    bool doctest_ok_ = true;                                                                   \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (...) {                                                                            \
      doctest_ok_ = false;                                                                     \
    }                                                                                          \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #expr);         \
  } while (0)

#define FAIL(msg)                                                                          \
  do {                                                                                     \
    ::doctest::detail::report_failure(__FILE__, __LINE__,                                  \
                                      std::string("FAIL: ") + ::doctest::detail::to_text(msg)); \
    throw ::doctest::detail::Abort{};                                                      \
  } while (0)
#define MESSAGE(msg) std::printf("    MESSAGE: %s\n", ::doctest::detail::to_text(msg).c_str())
#define CAPTURE(x) \
  const ::doctest::detail::Capture DOCTEST_UNIQUE(doctest_cap_)(std::string(#x " := ") + ::doctest::detail::to_text(x))
#define INFO(msg) const ::doctest::detail::Capture DOCTEST_UNIQUE(doctest_info_)(::doctest::detail::to_text(msg))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* filter = nullptr;
  const char* file_filter = nullptr;
  const char* exclude = nullptr;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--test-case=", 12) == 0) filter = argv[i] + 12;
    if (std::strncmp(argv[i], "--source-file=", 14) == 0) file_filter = argv[i] + 14;
    if (std::strncmp(argv[i], "--test-case-exclude=", 20) == 0) exclude = argv[i] + 20;
  }
  return ::doctest::run_all(filter, file_filter, exclude) == 0 ? 0 : 1;
}
#endif

#endif  // FOLP_TESTS_DOCTEST_SHIM_H_
