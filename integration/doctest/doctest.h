// TEST INFRASTRUCTURE ONLY. A restatement of the small doctest 2.x subset the reference's unit
// tests use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, INFO, doctest::Approx with epsilon /
// scale), so /root/reference/proj/tests/*.cpp compile unchanged here: the vendored doctest.h is
// git-ignored upstream (proj/.gitignore:2) and there is no network. Approx follows doctest's
// published rule: |lhs - v| < epsilon * (scale + max(|lhs|, |v|)), default epsilon =
// 100 * FLT_EPSILON, scale 1 (DOCTEST_EPSILON_FLOOR, an addition, raises every epsilon to a
// floor). Reporting: one line per failed assertion, a per-test-case verdict and a final summary;
// the exit status is the number of failed test cases (capped at 255).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double lhs) const {
        // DOCTEST_EPSILON_FLOOR (not in doctest): re-run the same assertions with every Approx
        // epsilon raised to at least this value (the north_star tolerance of the fp32 backend)
        static const double floor_eps = [] {
            const char* f = std::getenv("DOCTEST_EPSILON_FLOOR");
            return f ? std::atof(f) : 0.0;
        }();
        const double eps = std::fmax(epsilon_, floor_eps);
        return std::fabs(lhs - value_) < eps * (scale_ + std::fmax(std::fabs(lhs), std::fabs(value_)));
    }
    friend bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
    friend bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }
    friend bool operator!=(const Approx& a, double rhs) { return !a.matches(rhs); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || a.matches(lhs); }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || a.matches(lhs); }

private:
    double value_;
    double epsilon_ = static_cast<double>(FLT_EPSILON) * 100.0;
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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

struct State {
    long asserts = 0, failed_asserts = 0;
    long current_failed = 0;
    int printed = 0;
    std::string current;
};

inline State& state() {
    static State s;
    return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    ++s.current_failed;
    if (s.current_failed <= 3)  // first failures of a test case; the count is in the verdict
        std::printf("    %s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

inline int run_all() {
    State& s = state();
    int failed_cases = 0;
    const char* filter = std::getenv("DOCTEST_FILTER");
    int ran = 0;
    for (const TestCase& tc : registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++ran;
        s.current = tc.name;
        s.current_failed = 0;
        const long before = s.asserts;
        std::string err;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
            err = "REQUIRE failed";
        } catch (const std::exception& e) {
            err = std::string("unexpected exception: ") + e.what();
            ++s.current_failed;
        } catch (...) {
            err = "unexpected exception";
            ++s.current_failed;
        }
        const bool ok = s.current_failed == 0;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s  (%ld assertions, %ld failed)%s%s\n", ok ? "PASS" : "FAIL", tc.name,
                    s.asserts - before, s.current_failed, err.empty() ? "" : "  ", err.c_str());
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", ran, ran - failed_cases, failed_cases);
    std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", s.asserts, s.asserts - s.failed_asserts,
                s.failed_asserts);
    return failed_cases > 255 ? 255 : failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                            \
    static void fn();                                                                           \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_anon_test_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                 \
    do {                                                                                             \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                     \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);         \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                  \
    do {                                                                                            \
        bool doctest_thrown_ = false;                                                               \
        try {                                                                                       \
            static_cast<void>(expr);                                                                \
        } catch (const __VA_ARGS__&) {                                                              \
            doctest_thrown_ = true;                                                                 \
        } catch (...) {                                                                             \
        }                                                                                           \
        ::doctest::detail::report(doctest_thrown_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, \
                                  __LINE__);                                                        \
    } while (0)
#define INFO(...) static_cast<void>(0)
#define MESSAGE(...) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
