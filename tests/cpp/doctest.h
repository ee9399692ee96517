// doctest.h — a small from-scratch stand-in for the doctest macros the
// reference's unit tests use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, doctest::Approx), so proj/tests/test_engine.cpp and
// test_conv3d.cpp can be compiled unchanged against the GPU engine. The real
// doctest was never vendored into the reference. TEST ONLY.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
    int checks = 0, failed_checks = 0;
    bool current_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++state().checks;
    if (ok) return;
    ++state().failed_checks;
    state().current_failed = true;
    std::printf("  %s:%d: %s(%s) FAILED\n", file, line, fatal ? "REQUIRE" : "CHECK", expr);
    if (fatal) throw RequireFailed{};
}

// doctest::Approx: |lhs - value| < epsilon * (scale + max(|lhs|, |value|))
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

inline int run_all() {
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        state().current_failed = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("  unexpected exception: %s\n", e.what());
            state().current_failed = true;
        }
        std::printf("[%s] %s\n", state().current_failed ? "FAIL" : "PASS", tc.name);
        failed_cases += state().current_failed;
    }
    std::printf("test cases: %zu, failed: %d; checks: %d, failed: %d\n", registry().size(),
                failed_cases, state().checks, state().failed_checks);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                           \
    static void fn();                                                                   \
    static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                     \
    do {                                                                                \
        bool ok_ = false;                                                               \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const type&) {                                                         \
            ok_ = true;                                                                 \
        } catch (...) {                                                                 \
        }                                                                               \
        doctest::report(ok_, #expr " throws " #type, __FILE__, __LINE__, false);        \
    } while (0)
#define CHECK_NOTHROW(expr)                                                             \
    do {                                                                                \
        bool ok_ = true;                                                                \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (...) {                                                                 \
            ok_ = false;                                                                \
        }                                                                               \
        doctest::report(ok_, #expr " does not throw", __FILE__, __LINE__, false);       \
    } while (0)
