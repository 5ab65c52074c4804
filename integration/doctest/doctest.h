// doctest.h -- a minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include <doctest.h>, which is not
// in this image. This header implements the subset they use -- TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS, CHECK_THROWS_AS, doctest::Approx(...).epsilon(...), and the main() of
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so those files compile and run unmodified against the
// B200 operators (integration/gpu_operators.cpp). Semantics follow doctest: a failed CHECK is
// recorded and the case goes on, a failed REQUIRE ends the case, an exception escaping a case
// fails it; Approx compares |a - b| < eps * (scale + max(|a|, |b|)) with eps = 100 * FLT_EPSILON.
// Command line: -tc=<glob>[,<glob>..] runs only matching cases, -tce=<glob>[,..] skips matching ones.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    bool matches(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(value_)));
    }
    friend bool operator==(double x, const Approx& a) { return a.matches(x); }
    friend bool operator==(const Approx& a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
    friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }
    friend bool operator<=(double x, const Approx& a) { return x < a.value_ || a.matches(x); }
    friend bool operator>=(double x, const Approx& a) { return x > a.value_ || a.matches(x); }

private:
    double value_;
    double eps_ = 100.0 * FLT_EPSILON;
    double scale_ = 1.0;
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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct State {
    int failed_asserts = 0;
    int asserts = 0;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++state().asserts;
    if (ok) return;
    ++state().failed_asserts;
    std::printf("%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
}

inline bool glob(const char* p, const char* s) {
    if (!*p) return !*s;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    return *s && *p == *s && glob(p + 1, s + 1);
}

inline bool any_glob(const std::string& list, const char* s) {
    size_t i = 0;
    while (i <= list.size()) {
        size_t j = list.find(',', i);
        if (j == std::string::npos) j = list.size();
        if (glob(list.substr(i, j - i).c_str(), s)) return true;
        i = j + 1;
    }
    return false;
}

inline int run(int argc, char** argv) {
    std::string only, skip;
    for (int i = 1; i < argc; ++i) {
        if (!std::strncmp(argv[i], "-tc=", 4)) only = argv[i] + 4;
        if (!std::strncmp(argv[i], "-tce=", 5)) skip = argv[i] + 5;
    }
    int cases = 0, failed_cases = 0, skipped = 0;
    for (const Case& c : registry()) {
        if ((!only.empty() && !any_glob(only, c.name)) || (!skip.empty() && any_glob(skip, c.name))) {
            ++skipped;
            continue;
        }
        ++cases;
        const int before = state().failed_asserts;
        bool threw = false;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            threw = true;
            std::printf("%s:%d: ERROR: test case threw: %s\n", c.file, c.line, e.what());
        } catch (...) {
            threw = true;
            std::printf("%s:%d: ERROR: test case threw a non-std exception\n", c.file, c.line);
        }
        const bool ok = !threw && state().failed_asserts == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", cases, cases - failed_cases,
                failed_cases, skipped);
    std::printf("[doctest] assertions: %d | %d passed | %d failed\n", state().asserts,
                state().asserts - state().failed_asserts, state().failed_asserts);
    std::printf("[doctest] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                     \
    static void fn();                                                                        \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
    do {                                                                                          \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                 \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);     \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                              \
    } while (0)
#define CHECK_THROWS(...)                                                                         \
    do {                                                                                          \
        bool doctest_threw_ = false;                                                              \
        try {                                                                                     \
            static_cast<void>(__VA_ARGS__);                                                       \
        } catch (...) {                                                                           \
            doctest_threw_ = true;                                                                \
        }                                                                                         \
        ::doctest::detail::report(doctest_threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                \
    do {                                                                                          \
        bool doctest_threw_ = false;                                                              \
        try {                                                                                     \
            static_cast<void>(expr);                                                              \
        } catch (const __VA_ARGS__&) {                                                            \
            doctest_threw_ = true;                                                                \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::detail::report(doctest_threw_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);  \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
