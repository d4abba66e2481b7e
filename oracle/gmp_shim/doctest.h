// TEST INFRASTRUCTURE ONLY (oracle/).
//
// A small restatement of the doctest macros the reference's own test suites
// use (`/root/reference/proj/tests/*.cpp`: TEST_CASE, SUBCASE, CHECK*,
// REQUIRE, CHECK_THROWS_AS/WITH, CHECK_NOTHROW, MESSAGE, doctest::Approx).
// doctest itself is absent from the image; this lets
// oracle/Makefile build and run the reference's unit suites against the
// shim-compiled reference library, which pins the GMP shim before the
// oracle is trusted.  SUBCASE follows doctest/Catch "section" semantics: the
// test body is re-run until every leaf subcase has executed once.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <iostream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx &epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx &a) {
        double margin = a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
        return std::fabs(lhs - a.value_) < margin || lhs == a.value_;
    }
    friend bool operator==(const Approx &a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx &a) { return !(lhs == a); }

private:
    double value_;
    double eps_ = 1.1920929e-7 * 100; // doctest default: float epsilon * 100
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char *name;
    const char *file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase> &registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char *name, const char *file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RunState {
    std::set<std::vector<int>> completed;
    std::vector<int> stack;
    std::vector<bool> entered_at_depth;
    bool pending = false;
    std::vector<bool> child_pending;
    long failures = 0;
    long assertions = 0;
    std::string current;
};

inline RunState &state() {
    static RunState s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char *file, int line, const std::string &expr,
                   const std::string &extra = {}) {
    RunState &s = state();
    s.assertions++;
    if (ok) return;
    s.failures++;
    std::cerr << file << ":" << line << ": FAILED in '" << s.current << "': " << expr;
    if (!extra.empty()) std::cerr << " (" << extra << ")";
    std::cerr << "\n";
}

class Subcase {
public:
    Subcase(const char *, int line) {
        RunState &s = state();
        std::size_t depth = s.stack.size();
        if (s.entered_at_depth.size() <= depth) s.entered_at_depth.resize(depth + 1, false);
        std::vector<int> path = s.stack;
        path.push_back(line);
        if (s.completed.count(path)) return;
        if (s.entered_at_depth[depth]) {
            mark_pending();
            return;
        }
        s.entered_at_depth[depth] = true;
        s.stack.push_back(line);
        s.child_pending.push_back(false);
        if (s.entered_at_depth.size() <= depth + 1) s.entered_at_depth.resize(depth + 2, false);
        s.entered_at_depth[depth + 1] = false;
        entered_ = true;
    }
    ~Subcase() {
        if (!entered_) return;
        RunState &s = state();
        bool child_pending = s.child_pending.back();
        s.child_pending.pop_back();
        if (!child_pending) s.completed.insert(s.stack);
        s.stack.pop_back();
        if (child_pending) mark_pending();
    }
    explicit operator bool() const { return entered_; }

private:
    static void mark_pending() {
        RunState &s = state();
        s.pending = true;
        if (!s.child_pending.empty()) s.child_pending.back() = true;
    }
    bool entered_ = false;
};

inline int run_all() {
    RunState &s = state();
    int failed_cases = 0;
    for (const TestCase &tc : registry()) {
        s.completed.clear();
        s.current = tc.name;
        long before = s.failures;
        for (int guard = 0; guard < 10000; ++guard) {
            s.stack.clear();
            s.entered_at_depth.assign(1, false);
            s.child_pending.clear();
            s.pending = false;
            try {
                tc.fn();
            } catch (const RequireFailed &) {
            } catch (const std::exception &e) {
                report(false, tc.file, tc.line, "unexpected exception", e.what());
            }
            if (!s.pending) break;
        }
        if (s.failures != before) failed_cases++;
    }
    std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %ld | failures: %ld\n",
                registry().size(), failed_cases, s.assertions, s.failures);
    return failed_cases == 0 ? 0 : 1;
}

template <typename... Args>
std::string concat(const Args &...args) {
    std::ostringstream os;
    (os << ... << args);
    return os.str();
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(prefix) DOCTEST_CAT(prefix, __LINE__)

#define TEST_CASE_IMPL(fn, name)                                                                   \
    static void fn();                                                                              \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);      \
    static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_ANON(doctest_shim_tc_), name)

#define SUBCASE(name)                                                                              \
    if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_shim_sc_){name, __LINE__})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                               \
    do {                                                                                           \
        bool ok_ = static_cast<bool>(__VA_ARGS__);                                                 \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, #__VA_ARGS__);                          \
        if (!ok_) throw ::doctest::detail::RequireFailed{};                                        \
    } while (0)
#define CHECK_MESSAGE(cond, ...)                                                                   \
    ::doctest::detail::report(static_cast<bool>(cond), __FILE__, __LINE__, #cond,                  \
                              ::doctest::detail::concat(__VA_ARGS__))
#define MESSAGE(...) ((void)0)
#define CAPTURE(...) ((void)0)
#define FAIL_CHECK(...)                                                                            \
    do {                                                                                           \
        std::ostringstream os_;                                                                    \
        os_ << __VA_ARGS__;                                                                        \
        ::doctest::detail::report(false, __FILE__, __LINE__, "FAIL_CHECK", os_.str());             \
    } while (0)
#define CHECK_NOTHROW(...)                                                                         \
    do {                                                                                           \
        bool ok_ = true;                                                                           \
        try {                                                                                      \
            (void)(__VA_ARGS__);                                                                   \
        } catch (...) {                                                                            \
            ok_ = false;                                                                           \
        }                                                                                          \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, "nothrow: " #__VA_ARGS__);              \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool ok_ = false;                                                                          \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const __VA_ARGS__ &) {                                                            \
            ok_ = true;                                                                            \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, "throws_as: " #expr);                   \
    } while (0)
#define CHECK_THROWS_WITH(expr, msg)                                                               \
    do {                                                                                           \
        bool ok_ = false;                                                                          \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const std::exception &e_) {                                                       \
            ok_ = std::string(e_.what()) == std::string(msg);                                      \
        }                                                                                          \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, "throws_with: " #expr);                 \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
