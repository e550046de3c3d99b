// Minimal Catch2-compatible shim so the reference's unit suites
// (/root/reference/proj/tests/*_tests.cpp) can be compiled UNCHANGED against
// this repo's include/roundpipe headers (and against the reference headers,
// to validate the shim itself). Catch2 is not installed in this image.
// Supports TEST_CASE, CHECK/REQUIRE(+_FALSE), CHECK_THROWS_AS/REQUIRE_THROWS_AS,
// INFO and Catch::Approx(...).margin(...). Test infrastructure only.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct State {
  long checks = 0, failures = 0;
  std::vector<std::string> info;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireAbort {};
inline void record(bool ok, const char* expr, const char* file, int line,
                   bool fatal) {
  ++state().checks;
  if (ok) return;
  ++state().failures;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  for (const auto& m : state().info) std::fprintf(stderr, "    with: %s\n", m.c_str());
  if (fatal) throw RequireAbort{};
}
struct InfoScope {
  explicit InfoScope(std::string m) { state().info.push_back(std::move(m)); }
  ~InfoScope() { state().info.pop_back(); }
};
}  // namespace catch_shim

namespace Catch {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& margin(double m) { margin_ = m; return *this; }
  Approx& epsilon(double e) { eps_ = e; return *this; }
  friend bool operator==(double x, const Approx& a) { return a.eq(x); }
  friend bool operator==(const Approx& a, double x) { return a.eq(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.eq(x); }
 private:
  bool eq(double x) const {
    const double d = std::fabs(x - v_);
    return d <= margin_ || d <= eps_ * (1.0 + std::fmax(std::fabs(x), std::fabs(v_)));
  }
  double v_;
  double margin_ = 0.0;
  double eps_ = 1.1920929e-7f * 100;
};
}  // namespace Catch

#define CS_CAT2(a, b) a##b
#define CS_CAT(a, b) CS_CAT2(a, b)
#define TEST_CASE(...) CS_TEST_IMPL(CS_CAT(cs_test_, __LINE__), __VA_ARGS__)
#define CS_TEST_IMPL(fn, name, ...)                                   \
  static void fn();                                                   \
  static catch_shim::Registrar CS_CAT(fn, _reg)(name, &fn);           \
  static void fn()
#define CS_CHECK(expr, fatal) \
  catch_shim::record(static_cast<bool>(expr), #expr, __FILE__, __LINE__, fatal)
#define CHECK(...) CS_CHECK((__VA_ARGS__), false)
#define REQUIRE(...) CS_CHECK((__VA_ARGS__), true)
#define CHECK_FALSE(...) CS_CHECK(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) CS_CHECK(!(__VA_ARGS__), true)
#define CS_THROWS(expr, type, fatal)                                  \
  do {                                                                \
    bool cs_ok = false;                                               \
    try { (void)(expr); } catch (const type&) { cs_ok = true; } catch (...) {} \
    catch_shim::record(cs_ok, #expr " throws " #type, __FILE__, __LINE__, fatal); \
  } while (0)
#define CHECK_THROWS_AS(expr, type) CS_THROWS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) CS_THROWS(expr, type, true)
#define INFO(msg)                                                     \
  catch_shim::InfoScope CS_CAT(cs_info_, __LINE__)(                   \
      (static_cast<std::ostringstream&&>(std::ostringstream() << msg)).str())

int main() {
  int failed_cases = 0;
  for (const auto& c : catch_shim::registry()) {
    const long before = catch_shim::state().failures;
    try {
      c.fn();
    } catch (const catch_shim::RequireAbort&) {
    } catch (const std::exception& e) {
      ++catch_shim::state().failures;
      std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
    }
    if (catch_shim::state().failures != before) {
      ++failed_cases;
      std::fprintf(stderr, "test case FAILED: %s\n", c.name);
    }
  }
  std::printf("test cases: %zu | failed: %d | checks: %ld | failed checks: %ld\n",
              catch_shim::registry().size(), failed_cases,
              catch_shim::state().checks, catch_shim::state().failures);
  return failed_cases == 0 ? 0 : 1;
}
