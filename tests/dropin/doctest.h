// TEST INFRASTRUCTURE: a minimal doctest-compatible harness (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, CHECK_NOTHROW, doctest::Approx, doctest::Contains) — enough to compile the reference's
// own unit tests (proj/tests/test_{numerics,adapter,experts,memtier}.cpp) unmodified, against either the
// reference library or this repo's drop-in shim. The real doctest is not vendored in the reference.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    double value;
    double eps = 1.1920928955078125e-05 * 100;  // doctest's default: float epsilon * 100
};
inline bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {
struct Registry {
    std::vector<std::pair<const char*, void (*)()>> cases;
    static Registry& get() {
        static Registry r;
        return r;
    }
};
struct Registrar {
    Registrar(const char* name, void (*fn)()) { Registry::get().cases.emplace_back(name, fn); }
};
struct State {
    long asserts = 0, failed = 0;
    bool case_failed = false;
    static State& get() {
        static State s;
        return s;
    }
};
struct RequireFailure {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
    State& s = State::get();
    ++s.asserts;
    if (ok) return;
    ++s.failed;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    if (fatal) throw RequireFailure{};
}

inline int run_all() {
    auto& reg = Registry::get();
    int failed_cases = 0;
    for (auto& c : reg.cases) {
        State::get().case_failed = false;
        try {
            c.second();
        } catch (const RequireFailure&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "TEST CASE \"%s\" threw: %s\n", c.first, e.what());
            State::get().case_failed = true;
        } catch (...) {
            std::fprintf(stderr, "TEST CASE \"%s\" threw an unknown exception\n", c.first);
            State::get().case_failed = true;
        }
        if (State::get().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", c.first);
        }
    }
    std::printf("[doctest-mini] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
                reg.cases.size(), reg.cases.size() - size_t(failed_cases), failed_cases, State::get().asserts,
                State::get().failed);
    return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                   \
    static void fn();                                                                      \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                  \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                             \
        bool doctest_ok_ = false;                                                                    \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (const __VA_ARGS__&) {                                                               \
            doctest_ok_ = true;                                                                      \
        } catch (...) {                                                                              \
        }                                                                                            \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                          \
    do {                                                                                                  \
        bool doctest_ok_ = false;                                                                         \
        try {                                                                                             \
            (void)(expr);                                                                                 \
        } catch (const __VA_ARGS__& e_) {                                                                 \
            doctest_ok_ = (matcher).matches(e_.what());                                                   \
        } catch (...) {                                                                                   \
        }                                                                                                 \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                        \
    do {                                                                                           \
        bool doctest_ok_ = true;                                                                   \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (...) {                                                                            \
            doctest_ok_ = false;                                                                   \
        }                                                                                          \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
