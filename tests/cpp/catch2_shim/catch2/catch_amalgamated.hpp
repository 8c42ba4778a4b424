// catch_amalgamated.hpp -- TEST INFRASTRUCTURE ONLY.
//
// A minimal stand-in for the Catch2 v3 subset the reference's unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_NOTHROW, REQUIRE_THROWS,
// REQUIRE_THROWS_AS, REQUIRE_THROWS_WITH + ContainsSubstring, Catch::Approx),
// so that /root/reference/proj/tests/*.cpp compile UNCHANGED against the
// B200 drop-in header (Catch2 itself is not installed in this image).  The
// runner is tests/cpp/catch2_shim/catch_main.cpp.
#pragma once
#include <cmath>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
  std::string name;
  std::function<void()> fn;
  const char* file;
  int line;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, std::function<void()> fn, const char* file, int line) {
    registry().push_back({name, std::move(fn), file, line});
  }
};
struct Stats {
  long assertions = 0, failed = 0;
  bool case_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
struct RequireAbort {};
inline void report(bool ok, bool fatal, const char* expr, const char* file, int line,
                   const std::string& extra = {}) {
  ++stats().assertions;
  if (ok) return;
  ++stats().failed;
  stats().case_failed = true;
  std::printf("  FAILED %s:%d: %s%s%s\n", file, line, expr, extra.empty() ? "" : " -- ",
              extra.c_str());
  if (fatal) throw RequireAbort{};
}

// Approx (Catch2 v3 semantics: margin, or epsilon relative to the Approx's
// own value; default epsilon = 100 float epsilons).
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& margin(double m) { margin_ = m; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool equals(double x) const {
    const double d = std::fabs(x - v_);
    if (d <= margin_) return true;
    return d <= eps_ * (scale_ + (std::isinf(v_) ? 0.0 : std::fabs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.equals(x); }
  friend bool operator==(const Approx& a, double x) { return a.equals(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.equals(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.equals(x); }
  friend bool operator<=(double x, const Approx& a) { return x < a.v_ || a.equals(x); }
  friend bool operator>=(double x, const Approx& a) { return x > a.v_ || a.equals(x); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
  double scale_ = 0.0;
};

namespace Matchers {
struct ContainsSubstring {
  std::string s;
  explicit ContainsSubstring(std::string x) : s(std::move(x)) {}
  bool match(const std::string& what) const { return what.find(s) != std::string::npos; }
};
}  // namespace Matchers
inline bool throws_with(const std::string& what, const std::string& want) { return what == want; }
inline bool throws_with(const std::string& what, const Matchers::ContainsSubstring& m) {
  return m.match(what);
}

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                         \
  static void CATCH_SHIM_CAT(catch_shim_fn_, __LINE__)();                            \
  static ::Catch::Registrar CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)(               \
      name, &CATCH_SHIM_CAT(catch_shim_fn_, __LINE__), __FILE__, __LINE__);          \
  static void CATCH_SHIM_CAT(catch_shim_fn_, __LINE__)()

#define CATCH_SHIM_BOOL(expr, fatal, neg)                                            \
  do {                                                                               \
    bool ok_ = false;                                                                \
    std::string ex_;                                                                 \
    try {                                                                            \
      ok_ = static_cast<bool>(expr) != (neg);                                        \
    } catch (const ::Catch::RequireAbort&) {                                         \
      throw;                                                                         \
    } catch (const std::exception& e_) {                                             \
      ex_ = std::string("threw: ") + e_.what();                                      \
    }                                                                                \
    ::Catch::report(ok_, fatal, #expr, __FILE__, __LINE__, ex_);                     \
  } while (0)
#define CHECK(...) CATCH_SHIM_BOOL((__VA_ARGS__), false, false)
#define CHECK_FALSE(...) CATCH_SHIM_BOOL((__VA_ARGS__), false, true)
#define REQUIRE(...) CATCH_SHIM_BOOL((__VA_ARGS__), true, false)
#define REQUIRE_FALSE(...) CATCH_SHIM_BOOL((__VA_ARGS__), true, true)

#define REQUIRE_NOTHROW(...)                                                         \
  do {                                                                               \
    bool ok_ = true;                                                                 \
    std::string ex_;                                                                 \
    try {                                                                            \
      (void)(__VA_ARGS__);                                                           \
    } catch (const std::exception& e_) {                                             \
      ok_ = false;                                                                   \
      ex_ = e_.what();                                                               \
    }                                                                                \
    ::Catch::report(ok_, true, "REQUIRE_NOTHROW(" #__VA_ARGS__ ")", __FILE__, __LINE__, ex_); \
  } while (0)
#define REQUIRE_THROWS(...)                                                          \
  do {                                                                               \
    bool ok_ = false;                                                                \
    try {                                                                            \
      (void)(__VA_ARGS__);                                                           \
    } catch (...) {                                                                  \
      ok_ = true;                                                                    \
    }                                                                                \
    ::Catch::report(ok_, true, "REQUIRE_THROWS(" #__VA_ARGS__ ")", __FILE__, __LINE__); \
  } while (0)
#define REQUIRE_THROWS_AS(expr, Ex)                                                  \
  do {                                                                               \
    bool ok_ = false;                                                                \
    std::string got_ = "no exception";                                              \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const Ex&) {                                                            \
      ok_ = true;                                                                    \
    } catch (const std::exception& e_) {                                             \
      got_ = std::string("other exception: ") + e_.what();                           \
    } catch (...) {                                                                  \
      got_ = "non-std exception";                                                    \
    }                                                                                \
    ::Catch::report(ok_, true, "REQUIRE_THROWS_AS(" #expr ", " #Ex ")", __FILE__, __LINE__, \
                    ok_ ? std::string() : got_);                                     \
  } while (0)
#define REQUIRE_THROWS_WITH(expr, matcher)                                           \
  do {                                                                               \
    bool ok_ = false;                                                                \
    std::string got_ = "no exception";                                              \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const std::exception& e_) {                                             \
      got_ = e_.what();                                                              \
      ok_ = ::Catch::throws_with(got_, matcher);                                     \
    }                                                                                \
    ::Catch::report(ok_, true, "REQUIRE_THROWS_WITH(" #expr ")", __FILE__, __LINE__, got_); \
  } while (0)
