// Minimal stand-in for the subset of Catch2 v3 the reference's tests use
// (TEST_CASE, REQUIRE, REQUIRE_FALSE, REQUIRE_THROWS_AS, FAIL, INFO, Catch::Approx), so that
// /root/reference/proj/tests/*.cpp compile unmodified here (Catch2 is not installed,
// SURVEY §0.3). TEST INFRASTRUCTURE ONLY (oracle/_ref). Define CATCH_SHIM_MAIN in exactly
// one translation unit to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  std::function<void()> fn;
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
struct Failure {
  std::string what;
};
inline std::vector<std::string>& info_stack() {
  static std::vector<std::string> s;
  return s;
}
struct InfoScope {
  explicit InfoScope(std::string m) { info_stack().push_back(std::move(m)); }
  ~InfoScope() { info_stack().pop_back(); }
};
inline long& assertion_count() {
  static long n = 0;
  return n;
}
[[noreturn]] inline void fail(const char* file, int line, const std::string& msg) {
  std::ostringstream os;
  os << file << ":" << line << ": " << msg;
  for (const auto& s : info_stack()) os << "\n  with: " << s;
  throw Failure{os.str()};
}

// Catch2 v3 Approx: |a - v| <= margin  or  |a - v| <= epsilon * (scale + |v|)
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& margin(double m) { margin_ = m; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool matches(double a) const {
    const double d = std::fabs(a - v_);
    return d <= margin_ || d <= eps_ * (scale_ + std::fabs(std::isinf(v_) ? 0.0 : v_));
  }
  double value() const { return v_; }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
  double scale_ = 0.0;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& b, double a) { return b.matches(a); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }

inline int run_all() {
  int failed = 0;
  for (const auto& t : registry()) {
    try {
      t.fn();
    } catch (const Failure& f) {
      ++failed;
      std::printf("FAILED: %s\n  %s\n", t.name, f.what.c_str());
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAILED: %s\n  unexpected exception: %s\n", t.name, e.what());
    }
  }
  std::printf("%s: %zu test cases, %d failed, %ld assertions\n", failed ? "FAILED" : "All tests passed",
              registry().size(), failed, assertion_count());
  return failed ? 1 : 0;
}

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TC(fn, name)                                                            \
  static void fn();                                                                      \
  static ::Catch::Registrar CATCH_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);     \
  static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_TC(CATCH_SHIM_CAT(catch_shim_test_, __LINE__), name)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    ++::Catch::assertion_count();                                                     \
    if (!static_cast<bool>(__VA_ARGS__)) ::Catch::fail(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )"); \
  } while (0)
#define REQUIRE_FALSE(...)                                                            \
  do {                                                                                \
    ++::Catch::assertion_count();                                                     \
    if (static_cast<bool>(__VA_ARGS__)) ::Catch::fail(__FILE__, __LINE__, "REQUIRE_FALSE( " #__VA_ARGS__ " )"); \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                  \
  do {                                                                                \
    ++::Catch::assertion_count();                                                     \
    bool caught_ = false;                                                             \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const type&) {                                                           \
      caught_ = true;                                                                 \
    }                                                                                 \
    if (!caught_) ::Catch::fail(__FILE__, __LINE__, "REQUIRE_THROWS_AS( " #expr ", " #type " )"); \
  } while (0)
#define FAIL(msg)                                                                     \
  ::Catch::fail(__FILE__, __LINE__, [&] {                                             \
    std::ostringstream catch_shim_os_;                                                \
    catch_shim_os_ << "FAIL: " << msg;                                                \
    return catch_shim_os_.str();                                                      \
  }())
#define INFO(msg)                                                                     \
  ::Catch::InfoScope CATCH_SHIM_CAT(catch_shim_info_, __LINE__)(                        \
      [&] {                                                                           \
        std::ostringstream catch_shim_os_;                                            \
        catch_shim_os_ << msg;                                                        \
        return catch_shim_os_.str();                                                  \
      }())

#ifdef CATCH_SHIM_MAIN
int main() { return ::Catch::run_all(); }
#endif
