// Minimal doctest-compatible test harness (doctest.h is not vendored in the
// reference tree and there is no network). Covers the surface the reference
// unit tests use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, CAPTURE, FAIL, doctest::Approx(.epsilon),
// doctest::Contains and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || a == b; }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || a == b; }

 private:
  double v_;
  double eps_ = 1e-5 * 100;  // doctest default: float epsilon * 100
};

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  bool matches(const std::string& msg) const { return msg.find(s) != std::string::npos; }
};
inline bool message_matches(const Contains& c, const std::string& m) { return c.matches(m); }
inline bool message_matches(const char* s, const std::string& m) { return m == s; }
inline bool message_matches(const std::string& s, const std::string& m) { return m == s; }

namespace detail {
struct TestCase {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct Abort {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline std::vector<std::string>& captures() {
  static std::vector<std::string> c;
  return c;
}
inline void report(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
  for (const auto& c : captures()) std::fprintf(stderr, "    with %s\n", c.c_str());
}
struct CaptureGuard {
  CaptureGuard(std::string s) { captures().push_back(std::move(s)); }
  ~CaptureGuard() { captures().pop_back(); }
};
template <class T>
std::string to_s(const T& v) {
  std::ostringstream os;
  os << v;
  return os.str();
}
inline int run_all() {
  int failed_cases = 0;
  for (auto& tc : registry()) {
    int before = failures();
    try {
      tc.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      report("<test>", 0, std::string("unexpected exception in \"") + tc.name + "\": " + e.what());
    }
    if (failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d\n",
              registry().size(), registry().size() - failed_cases, failed_cases, checks());
  return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                              \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                  \
  static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(            \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...)                                                                          \
  do {                                                                                      \
    ++::doctest::detail::checks();                                                          \
    try {                                                                                   \
      if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )"); \
    } catch (const std::exception& e) {                                                     \
      ::doctest::detail::report(__FILE__, __LINE__,                                         \
                                std::string("CHECK( " #__VA_ARGS__ " ) threw: ") + e.what()); \
    }                                                                                       \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    ++::doctest::detail::checks();                                                         \
    if (!(__VA_ARGS__)) {                                                                  \
      ::doctest::detail::report(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");       \
      throw ::doctest::detail::Abort{};                                                    \
    }                                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    ++::doctest::detail::checks();                                                          \
    bool doctest_ok_ = false;                                                               \
    try {                                                                                   \
      (void)(expr);                                                                         \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_ok_ = true;                                                                   \
    } catch (...) {                                                                         \
    }                                                                                       \
    if (!doctest_ok_)                                                                       \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                \
  do {                                                                                      \
    ++::doctest::detail::checks();                                                          \
    bool doctest_ok_ = false;                                                               \
    try {                                                                                   \
      (void)(expr);                                                                         \
    } catch (const __VA_ARGS__& e) {                                                        \
      doctest_ok_ = ::doctest::message_matches(msg, std::string(e.what()));                 \
    } catch (...) {                                                                         \
    }                                                                                       \
    if (!doctest_ok_)                                                                       \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS( " #expr " )");   \
  } while (0)
#define CAPTURE(x) \
  ::doctest::detail::CaptureGuard DOCTEST_CAT(doctest_cap_, __LINE__)(std::string(#x " := ") + ::doctest::detail::to_s(x))
#define FAIL(msg)                                                                   \
  do {                                                                              \
    ::doctest::detail::report(__FILE__, __LINE__, std::string("FAIL: ") + (msg));   \
    throw ::doctest::detail::Abort{};                                               \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
