// Minimal stand-in for doctest (the reference's unit suites include <doctest.h>, which
// /root/reference does not ship).  Implements exactly what proj/tests/unit_capi.cpp
// uses: TEST_CASE registration, CHECK / REQUIRE, doctest::Approx and a main() with
// doctest's -tce=<name>[,<name>...] test-case exclusion.  Failures are reported with
// file:line and the expression text; the exit status is the number of failed cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    double value;
    double eps = 1.1920928955078125e-07 * 100;  // doctest's default epsilon (float eps * 100)
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) < a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
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
struct Reg {
    Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline int& failures() {
    static int f = 0;
    return f;
}
struct RequireFailed {};
inline void fail(const char* kind, const char* expr, const char* file, int line) {
    ++failures();
    std::printf("%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                   \
    static void fn();                                                             \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn);               \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                                        \
    do {                                                                                  \
        if (!(__VA_ARGS__)) ::doctest::detail::fail("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define REQUIRE(...)                                                                          \
    do {                                                                                      \
        if (!(__VA_ARGS__)) {                                                                 \
            ::doctest::detail::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);             \
            throw ::doctest::detail::RequireFailed{};                                         \
        }                                                                                     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> exclude;
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        const char* p = std::strncmp(a, "-tce=", 5) == 0 ? a + 5 : nullptr;
        if (!p) continue;
        std::string s(p);
        std::size_t pos = 0;
        while (pos <= s.size()) {
            const std::size_t c = s.find(',', pos);
            exclude.push_back(s.substr(pos, c == std::string::npos ? std::string::npos : c - pos));
            if (c == std::string::npos) break;
            pos = c + 1;
        }
    }
    int failed_cases = 0, run = 0, skipped = 0;
    for (auto& c : ::doctest::detail::registry()) {
        bool skip = false;
        for (auto& e : exclude) skip |= e == c.name;
        if (skip) {
            ++skipped;
            continue;
        }
        ++run;
        const int before = ::doctest::detail::failures();
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (...) {
            ::doctest::detail::fail("TEST_CASE", "unexpected exception", c.name, 0);
        }
        const bool bad = ::doctest::detail::failures() != before;
        failed_cases += bad;
        std::printf("[%s] %s\n", bad ? "FAIL" : " ok ", c.name);
    }
    std::printf("test cases: %d run, %d failed, %d skipped; assertions failed: %d\n", run, failed_cases, skipped,
                ::doctest::detail::failures());
    return failed_cases;
}
#endif
