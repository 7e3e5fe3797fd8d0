// doctest.h — a minimal stand-in for the doctest macros the reference's unit
// tests use (TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS, REQUIRE,
// doctest::Approx(...).epsilon(...)). doctest itself is not in this image;
// this header lets integration/Makefile compile the reference's own tests
// (/root/reference/proj/tests/*.cpp, unmodified) twice — against the reference
// alone and with the hot path resolved to the B200 shim — so
// tests/test_integration.py can compare the per-test outcomes.
//
// Test infrastructure only. Approx follows doctest's published comparison:
// |lhs - v| < eps * (scale + max(|lhs|, |v|)), eps = 100 * FLT_EPSILON and
// scale = 1 by default.
//
// Output, one line per test case: "TEST <PASS|FAIL> <file>:<line> <name>",
// each failed assertion on its own "  fail <file>:<line> <expr>" line, and a
// final "SUMMARY <cases> <failed cases> <assertions> <failed assertions>".
// Exit code 0 iff every test case passed. argv[1], when given, is a substring
// filter on test-case names.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value)
        : eps_(double(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0), value_(value) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
    friend bool operator<(double lhs, const Approx& a) { return lhs < a.value_ && !(lhs == a); }
    friend bool operator>(double lhs, const Approx& a) { return lhs > a.value_ && !(lhs == a); }

private:
    double eps_, scale_, value_;
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

struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct Counters {
    long asserts = 0, failed = 0;
};

inline Counters& counters() {
    static Counters c;
    return c;
}

struct RequireAbort {};

inline const char* base(const char* f) {
    const char* s = std::strrchr(f, '/');
    return s ? s + 1 : f;
}

inline void report(bool ok, const char* file, int line, const char* expr, bool require) {
    ++counters().asserts;
    if (ok) return;
    ++counters().failed;
    std::printf("  fail %s:%d %s\n", base(file), line, expr);
    if (require) throw RequireAbort{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, reg, name)                                                 \
    static void fn();                                                              \
    static const ::doctest::detail::Reg reg(name, __FILE__, __LINE__, &fn);       \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_fn_, __COUNTER__), DOCTEST_CAT(doctest_reg_, __COUNTER__), name)

#define DOCTEST_ASSERT_(cond, text, require)                                                       \
    do {                                                                                           \
        bool doctest_ok_ = false;                                                                  \
        try {                                                                                      \
            doctest_ok_ = static_cast<bool>(cond);                                                 \
        } catch (const ::doctest::detail::RequireAbort&) {                                         \
            throw;                                                                                 \
        } catch (...) {                                                                            \
            doctest_ok_ = false;                                                                   \
        }                                                                                          \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, text, require);                 \
    } while (0)
#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, type)                                                                \
    do {                                                                                           \
        bool doctest_ok_ = false;                                                                  \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const type&) {                                                                    \
            doctest_ok_ = true;                                                                    \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "throws " #type ": " #expr, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    using namespace doctest::detail;
    const char* filter = argc > 1 ? argv[1] : nullptr;
    long cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++cases;
        const long before = counters().failed;
        bool threw = false;
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            threw = true;
            std::printf("  fail %s:%d unexpected exception: %s\n", base(c.file), c.line, e.what());
        } catch (...) {
            threw = true;
            std::printf("  fail %s:%d unexpected exception\n", base(c.file), c.line);
        }
        const bool ok = !threw && counters().failed == before;
        if (!ok) ++failed_cases;
        std::printf("TEST %s %s:%d %s\n", ok ? "PASS" : "FAIL", base(c.file), c.line, c.name);
        std::fflush(stdout);
    }
    std::printf("SUMMARY %ld %ld %ld %ld\n", cases, failed_cases, counters().asserts, counters().failed);
    return failed_cases ? 1 : 0;
}
#endif
