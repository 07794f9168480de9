// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (proj/tests/test_*.cpp) are written against
// doctest, whose header is not vendored with the reference (vendor/ is
// git-ignored, proj/.gitignore:2). This shim implements the subset they use
// -- TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS,
// doctest::Approx (epsilon/scale with doctest's comparison rule) and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so those files compile unmodified
// against include/topoopt/*.hpp and run against libtopoopt_b200.so.
//
// Runner: `binary [substring]` runs every test case (or those whose name
// contains the substring) and prints one line per failed assertion plus a
// summary; the exit code is the number of failed test cases (capped at 255).
#pragma once

#include <algorithm>
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
    // doctest's rule: |lhs - v| < eps (scale + max(|lhs|, |v|))
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

   private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
inline bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value() || rhs.matches(lhs); }
inline bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value() || rhs.matches(lhs); }

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
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline void fail(const char* file, int line, const char* what, const char* expr) {
    ++state().failed_checks;
    state().case_failed = true;
    std::printf("%s:%d: FAILED %s( %s )\n", file, line, what, expr);
}

inline bool check(bool ok, const char* file, int line, const char* what, const char* expr) {
    ++state().checks;
    if (!ok) fail(file, line, what, expr);
    return ok;
}

inline int run(int argc, char** argv) {
    const char* filter = nullptr;
    for (int k = 1; k < argc; ++k)
        if (argv[k][0] != '-') filter = argv[k];
    int cases = 0, failed_cases = 0;
    for (const TestCase& tc : registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++cases;
        state().case_failed = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("%s:%d: FAILED test case threw: %s\n", tc.file, tc.line, e.what());
            state().case_failed = true;
        } catch (...) {
            std::printf("%s:%d: FAILED test case threw a non-standard exception\n", tc.file, tc.line);
            state().case_failed = true;
        }
        if (state().case_failed) {
            ++failed_cases;
            std::printf("  in TEST_CASE \"%s\"\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases,
                failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", state().checks,
                state().checks - state().failed_checks, state().failed_checks);
    std::fflush(stdout);
    return std::min(failed_cases, 255);
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                          \
    static void fn();                                                                         \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ((void)::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__))
#define CHECK_FALSE(...) \
    ((void)::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__))
#define REQUIRE(...)                                                                                      \
    do {                                                                                                  \
        if (!::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__)) \
            throw ::doctest::detail::RequireFailed{};                                                     \
    } while (0)
#define REQUIRE_FALSE(...)                                                                                 \
    do {                                                                                                   \
        if (!::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE_FALSE", \
                                      #__VA_ARGS__))                                                       \
            throw ::doctest::detail::RequireFailed{};                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                    \
    do {                                                                                              \
        bool threw_ = false;                                                                          \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const __VA_ARGS__&) {                                                                \
            threw_ = true;                                                                            \
        } catch (...) {                                                                               \
        }                                                                                             \
        ::doctest::detail::check(threw_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
