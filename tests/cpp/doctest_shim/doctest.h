// Minimal doctest-compatible test runner (written for this repo; the real
// doctest.h is not in the image).  Supports the subset the reference's
// planner suite uses: TEST_CASE, SUBCASE (run inline as a block), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, FAIL and doctest::Approx.
// Used by tests/test_reference_suite.py to run proj/tests/*.cpp (compiled
// straight from /root/reference) against libepp_planner.so.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    bool matches(double other) const {
        return std::fabs(other - value_) <
               eps_ * (1.0 + std::max(std::fabs(other), std::fabs(value_)));
    }
private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default scale
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

namespace shim {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
struct Registrar {
    Registrar(const char* n, void (*f)(), const char* file, int line) {
        registry().push_back({n, f, file, line});
    }
};
struct Abort {};
inline long& checks() { static long c = 0; return c; }
inline long& failures() { static long f = 0; return f; }
inline void fail(const char* file, int line, const std::string& what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}
inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        const long before = failures();
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            fail(c.file, c.line, "unexpected non-std exception");
        }
        if (failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %ld | failed checks: %ld\n",
                registry().size(), registry().size() - failed_cases, failed_cases, checks(),
                failures());
    return failed_cases == 0 ? 0 : 1;
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(base) DOCTEST_CAT(base, __LINE__)

#define TEST_CASE(name)                                                                  \
    static void DOCTEST_UNIQUE(doctest_case_)();                                          \
    static ::doctest::shim::Registrar DOCTEST_UNIQUE(doctest_reg_)(                       \
        name, &DOCTEST_UNIQUE(doctest_case_), __FILE__, __LINE__);                        \
    static void DOCTEST_UNIQUE(doctest_case_)()

#define SUBCASE(name) if (const char* doctest_subcase_ = (name); doctest_subcase_ != nullptr)

#define DOCTEST_CHECK_IMPL(cond, text, abort)                                             \
    do {                                                                                  \
        ++::doctest::shim::checks();                                                      \
        if (!(cond)) {                                                                    \
            ::doctest::shim::fail(__FILE__, __LINE__, text);                             \
            if (abort) throw ::doctest::shim::Abort{};                                    \
        }                                                                                 \
    } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), "CHECK(" #__VA_ARGS__ ")", false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), "CHECK_FALSE(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), "REQUIRE(" #__VA_ARGS__ ")", true)

#define CHECK_THROWS_AS(expr, ...)                                                        \
    do {                                                                                  \
        ++::doctest::shim::checks();                                                      \
        bool doctest_ok_ = false;                                                         \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (const __VA_ARGS__&) {                                                    \
            doctest_ok_ = true;                                                           \
        } catch (...) {                                                                   \
        }                                                                                 \
        if (!doctest_ok_)                                                                 \
            ::doctest::shim::fail(__FILE__, __LINE__,                                     \
                                  "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")");        \
    } while (0)

#define FAIL(msg)                                                                         \
    do {                                                                                  \
        std::ostringstream doctest_os_;                                                   \
        doctest_os_ << msg;                                                               \
        ::doctest::shim::fail(__FILE__, __LINE__, doctest_os_.str());                    \
        throw ::doctest::shim::Abort{};                                                   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
