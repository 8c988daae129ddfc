// Minimal doctest-compatible shim (TEST INFRASTRUCTURE).  The reference's unit
// tests include <doctest.h> from its vendor/ tree, which is not part of the
// reference snapshot; this header provides the subset they use (TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS, CHECK_NOTHROW,
// FAIL, doctest::Approx) so that those test files compile UNMODIFIED against
// this repository's sgl:: mirror (include/sgl/*.hpp).  Output: one line per
// failed check, a summary line, exit status = number of failed test cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <map>
#include <sstream>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default: float epsilon * 100
    double scale_ = 1.0;
};

namespace detail {

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

struct Abort {};  // a failed REQUIRE ends the test case

inline int& failed_checks() {
    static int n = 0;
    return n;
}
inline const char*& current_case() {
    static const char* c = "";
    return c;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    if (ok) return;
    ++failed_checks();
    std::printf("  FAILED %s: %s (%s:%d)\n", current_case(), expr, file, line);
    if (fatal) throw Abort{};
}

inline int run_all() {
    int failed_cases = 0, passed = 0;
    for (const Case& c : registry()) {
        current_case() = c.name;
        const int before = failed_checks();
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            ++failed_checks();
            std::printf("  FAILED %s: unexpected exception: %s\n", c.name, e.what());
        }
        const bool ok = failed_checks() == before;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
        if (ok) ++passed;
        else ++failed_cases;
    }
    std::printf("[doctest shim] test cases: %d passed, %d failed; failed checks: %d\n", passed, failed_cases,
                failed_checks());
    return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                             \
    static void fn();                                                                \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);              \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg)                                                                    \
    do {                                                                             \
        std::ostringstream doctest_os_;                                              \
        doctest_os_ << msg;                                                          \
        doctest::detail::report(false, doctest_os_.str().c_str(), __FILE__, __LINE__, true); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
    do {                                                                             \
        bool doctest_ok_ = false;                                                    \
        try {                                                                        \
            static_cast<void>(expr);                                                 \
        } catch (const __VA_ARGS__&) {                                               \
            doctest_ok_ = true;                                                      \
        } catch (...) {                                                              \
        }                                                                            \
        doctest::detail::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS(expr)                                                           \
    do {                                                                             \
        bool doctest_ok_ = false;                                                    \
        try {                                                                        \
            static_cast<void>(expr);                                                 \
        } catch (...) {                                                              \
            doctest_ok_ = true;                                                      \
        }                                                                            \
        doctest::detail::report(doctest_ok_, #expr " throws", __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                          \
    do {                                                                             \
        bool doctest_ok_ = true;                                                     \
        try {                                                                        \
            static_cast<void>(expr);                                                 \
        } catch (...) {                                                              \
            doctest_ok_ = false;                                                     \
        }                                                                            \
        doctest::detail::report(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
