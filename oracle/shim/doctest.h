// Minimal doctest-compatible test shim (test infrastructure only).
//
// The reference keeps doctest under a git-ignored vendor/ directory that is
// absent from /root/reference (proj/.gitignore:2, proj/CMakeLists.txt:10), so
// its unit tests (proj/tests/*.cpp) cannot be built as shipped.  This header
// implements the subset of the doctest surface those files use -- TEST_CASE,
// CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx and
// doctest::Contains -- so the reference's own test sources compile unchanged
// against (a) the reference library (oracle/_ref) and (b) this repo's drop-in
// library.  It is never linked into the product.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value, eps = 1.1920929e-7 * 100, scale_ = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    bool matches(double other) const {
        double m = std::fmax(std::fabs(other), std::fabs(value));
        return std::fabs(other - value) < eps * (scale_ + m);
    }
};
template <class T> bool operator==(T lhs, const Approx& a) { return a.matches((double)lhs); }
template <class T> bool operator==(const Approx& a, T rhs) { return a.matches((double)rhs); }
template <class T> bool operator!=(T lhs, const Approx& a) { return !a.matches((double)lhs); }

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool check(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};
struct RequireFailed {};
inline long& assertions() { static long n = 0; return n; }
inline long& failures() { static long n = 0; return n; }
inline const char*& current() { static const char* c = ""; return c; }
inline void fail(const char* expr, const char* file, int line) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED in [%s]: %s\n", file, line, current(), expr);
}
inline bool match_msg(const char* m, const char* want) { return std::string(m) == want; }
inline bool match_msg(const char* m, const Contains& c) { return c.check(m); }
inline int run_all() {
    int failedCases = 0;
    for (const Case& c : registry()) {
        current() = c.name;
        long before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::fprintf(stderr, "%s:%d: [%s] threw: %s\n", c.file, c.line, c.name, e.what());
        }
        if (failures() != before) ++failedCases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
                registry().size(), registry().size() - failedCases, failedCases, assertions(),
                failures());
    return failedCases ? 1 : 0;
}
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                          \
    static void fn();                                                                      \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_IMPL(expr, fatal)                                                   \
    do {                                                                                   \
        ++::doctest::detail::assertions();                                                 \
        if (!(expr)) {                                                                     \
            ::doctest::detail::fail(#expr, __FILE__, __LINE__);                            \
            if (fatal) throw ::doctest::detail::RequireFailed{};                           \
        }                                                                                  \
    } while (0)
#define CHECK(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, type)                                                        \
    do {                                                                                   \
        ++::doctest::detail::assertions();                                                 \
        bool caught_ = false;                                                              \
        try { (void)(expr); } catch (const type&) { caught_ = true; } catch (...) {}       \
        if (!caught_) ::doctest::detail::fail(#expr " throws " #type, __FILE__, __LINE__); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, type)                                              \
    do {                                                                                   \
        ++::doctest::detail::assertions();                                                 \
        bool ok_ = false;                                                                  \
        try { (void)(expr); } catch (const type& e_) {                                     \
            ok_ = ::doctest::detail::match_msg(e_.what(), msg);                            \
        } catch (...) {}                                                                   \
        if (!ok_) ::doctest::detail::fail(#expr " throws " #type " with message", __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
