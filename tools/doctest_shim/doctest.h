// Minimal doctest-compatible test harness (own implementation) used to compile
// the reference's test suites (/root/reference/proj/tests, which expect the
// absent vendor/doctest.h) against this library.  Supports TEST_CASE,
// SUBCASE (each leaf subcase runs in its own pass of the test body), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
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
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

  private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct State {
    int target = 0;       // leaf subcase executed in this pass
    int seen = 0;         // subcases met so far in this pass
    int entered = -1;     // subcase index currently open (no nesting support needed)
    long checks = 0;
    long failures = 0;
    bool case_failed = false;
};

inline State& st() {
    static State s;
    return s;
}

struct Register {
    Register(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};

struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++st().checks;
    if (ok) return;
    ++st().failures;
    st().case_failed = true;
    std::printf("%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

struct Subcase {
    bool run;
    explicit Subcase(const char*) {
        State& s = st();
        run = s.entered < 0 && s.seen == s.target;
        if (run) s.entered = s.seen;
        ++s.seen;
    }
    ~Subcase() {
        if (run) st().entered = -1;
    }
    explicit operator bool() const { return run; }
};

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        State& s = st();
        s.case_failed = false;
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            s.entered = -1;
            try {
                c.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                std::printf("%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
                s.case_failed = true;
                ++s.failures;
            }
            if (s.target + 1 >= s.seen) break;  // every leaf subcase ran
        }
        if (s.case_failed) {
            ++failed_cases;
            std::printf("[case FAILED] %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %ld | %ld failed\n",
                registry().size(), failed_cases, st().checks, st().failures);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                               \
    static void fn();                                                                            \
    static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);     \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(sc_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                             \
    do {                                                                                         \
        const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                                  \
        ::doctest::detail::report(doctest_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);      \
        if (!doctest_ok) throw ::doctest::detail::RequireAbort{};                                \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                              \
    do {                                                                                         \
        bool doctest_thrown = false;                                                             \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (const type&) {                                                                  \
            doctest_thrown = true;                                                               \
        } catch (...) {                                                                          \
        }                                                                                        \
        ::doctest::detail::report(doctest_thrown, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                      \
    do {                                                                                         \
        bool doctest_ok = true;                                                                  \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (...) {                                                                          \
            doctest_ok = false;                                                                  \
        }                                                                                        \
        ::doctest::detail::report(doctest_ok, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);       \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
