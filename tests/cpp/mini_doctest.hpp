// Minimal doctest-compatible subset (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx) -- the reference's tests use doctest.h, which is not vendored
// (proj/.gitignore:2).  Enough to port proj/tests/test_optim.cpp checks 1:1.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 1e-5;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v) <= b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v)));
  }
};
struct Registry {
  std::vector<std::pair<std::string, std::function<void()>>> cases;
  int failed = 0, checks = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};
struct Reg {
  Reg(const char* n, std::function<void()> f) { Registry::get().cases.emplace_back(n, f); }
};
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_CASE(name)                                                   \
  static void DT_CAT(dt_fn_, __LINE__)();                                 \
  static doctest::Reg DT_CAT(dt_reg_, __LINE__)(name, DT_CAT(dt_fn_, __LINE__)); \
  static void DT_CAT(dt_fn_, __LINE__)()
#define CHECK(expr)                                                               \
  do {                                                                            \
    ++doctest::Registry::get().checks;                                            \
    if (!(expr)) {                                                                \
      ++doctest::Registry::get().failed;                                          \
      std::printf("%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #expr);        \
    }                                                                             \
  } while (0)
#define REQUIRE(expr) CHECK(expr)
#define CHECK_THROWS_AS(expr, type)                                                   \
  do {                                                                                \
    ++doctest::Registry::get().checks;                                                \
    bool ok_ = false;                                                                 \
    try {                                                                             \
      expr;                                                                           \
    } catch (const type&) {                                                           \
      ok_ = true;                                                                     \
    } catch (...) {                                                                   \
    }                                                                                 \
    if (!ok_) {                                                                       \
      ++doctest::Registry::get().failed;                                              \
      std::printf("%s:%d: CHECK_THROWS_AS(%s, %s) failed\n", __FILE__, __LINE__, #expr, #type); \
    }                                                                                 \
  } while (0)

inline int doctest_main() {
  auto& r = doctest::Registry::get();
  for (auto& [name, fn] : r.cases) {
    const int before = r.failed;
    try {
      fn();
    } catch (const std::exception& e) {
      ++r.failed;
      std::printf("test case '%s' threw: %s\n", name.c_str(), e.what());
    }
    std::printf("[%s] %s\n", r.failed == before ? "ok" : "FAIL", name.c_str());
  }
  std::printf("%zu test cases, %d checks, %d failed\n", r.cases.size(), r.checks, r.failed);
  return r.failed ? 1 : 0;
}
