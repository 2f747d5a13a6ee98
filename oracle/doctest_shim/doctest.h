// Test-only doctest-compatible shim — ORACLE INFRASTRUCTURE.
//
// The reference's unit suites (/root/reference/proj/tests/*.cpp) use doctest,
// which is git-ignored upstream (proj/.gitignore:2) and absent here. This
// header implements the macro subset those suites use (TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW, REQUIRE, FAIL, INFO,
// doctest::Approx) so the UNMODIFIED suites run against the Eigen shim and
// validate it (oracle/Makefile `ref-tests`).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

private:
    double value_;
    double epsilon_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
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

struct State {
    long checks = 0;
    long failures = 0;
    bool current_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline int register_test(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
    return 0;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++state().checks;
    if (!ok) {
        ++state().failures;
        state().current_failed = true;
        std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    }
}

inline int run_all() {
    int failed_cases = 0;
    const char* filter = std::getenv("DOCTEST_FILTER");
    for (const auto& tc : registry()) {
        if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
        state().current_failed = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++state().failures;
            state().current_failed = true;
            std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
        }
        if (state().current_failed) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %ld | %ld failed\n",
                registry().size(), failed_cases, state().checks, state().failures);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                          \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                            \
    static const int DOCTEST_CAT(doctest_reg_, __LINE__) = doctest::detail::register_test(      \
        name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                          \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
    do {                                                                                          \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                  \
        doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);        \
        if (!doctest_ok_) throw doctest::detail::RequireFailed{};                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                \
    do {                                                                                          \
        bool doctest_ok_ = false;                                                                 \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const __VA_ARGS__&) {                                                            \
            doctest_ok_ = true;                                                                   \
        } catch (...) {                                                                           \
        }                                                                                         \
        doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);       \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                       \
    do {                                                                                          \
        bool doctest_ok_ = true;                                                                  \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (...) {                                                                           \
            doctest_ok_ = false;                                                                  \
        }                                                                                         \
        doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);         \
    } while (0)
#define FAIL(msg)                                                                                 \
    do {                                                                                          \
        doctest::detail::report(false, "FAIL", "", __FILE__, __LINE__);                           \
        throw doctest::detail::RequireFailed{};                                                   \
    } while (0)
#define INFO(...) ((void)0)
#define MESSAGE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
