// Minimal Catch2-v3-compatible shim (TEST INFRASTRUCTURE ONLY) so the
// reference's own unit tests (/root/reference/proj/tests/unit/*.cpp) compile
// and run unmodified: the vendored Catch2 they include is absent
// (proj/.gitignore:2).  Supports exactly what those files use: TEST_CASE,
// SECTION, REQUIRE, REQUIRE_THAT + Matchers::WithinAbs, REQUIRE_THROWS_AS.
// SECTIONs run inline in one pass (the reference's sections are independent).
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace catch_shim {
struct Case { const char* name; const char* file; int line; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline long& checks() { static long c = 0; return c; }
struct Registrar { Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); } };
struct Failure { std::string what; };
[[noreturn]] inline void fail(const char* expr, const char* file, int line) {
    char buf[1024];
    std::snprintf(buf, sizeof buf, "%s:%d: REQUIRE(%s) failed", file, line, expr);
    throw Failure{buf};
}
}  // namespace catch_shim

namespace Catch { namespace Matchers {
struct WithinAbs {
    double target, eps;
    WithinAbs(double t, double e) : target(t), eps(e) {}
    bool match(double v) const { return std::fabs(v - target) <= eps; }
};
}}  // namespace Catch::Matchers

#define CS_CAT2(a, b) a##b
#define CS_CAT(a, b) CS_CAT2(a, b)
#define CS_TEST_CASE2(fn, name)                                                          \
    static void fn();                                                                    \
    static catch_shim::Registrar CS_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);       \
    static void fn()
#define TEST_CASE(name, ...) CS_TEST_CASE2(CS_CAT(cs_test_, __COUNTER__), name)
#define SECTION(name) if (true)
#define REQUIRE(...)                                                                     \
    do {                                                                                 \
        ++catch_shim::checks();                                                          \
        if (!(__VA_ARGS__)) catch_shim::fail(#__VA_ARGS__, __FILE__, __LINE__);          \
    } while (0)
#define REQUIRE_THAT(arg, matcher)                                                       \
    do {                                                                                 \
        ++catch_shim::checks();                                                          \
        if (!(matcher).match(arg)) catch_shim::fail(#arg " matches " #matcher, __FILE__, __LINE__); \
    } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                    \
    do {                                                                                 \
        ++catch_shim::checks();                                                          \
        bool cs_ok = false;                                                              \
        try { (void)(expr); } catch (const type&) { cs_ok = true; } catch (...) {}      \
        if (!cs_ok) catch_shim::fail(#expr " throws " #type, __FILE__, __LINE__);        \
    } while (0)
